#!/bin/bash
# tools/profile_round.sh PREFIX: bench line, ncu launch list of the bench step, ncu --set full
# of the build / merge / classify kernels on the headline workload, all-config sweep.
# Run on the GPU box (gpurun); outputs under gpurun_out/PREFIX_*.
P=${1:-prof}
O=gpurun_out
mkdir -p $O
timeout 400 python bench.py > $O/${P}_bench.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_times.py $O/${P}_launches.csv > $O/${P}_launch_times.txt
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"k_build_flat|k_merge_fused" -c 2 \
  -o $O/${P}_build python tools/kbench.py model --scene c3 > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:k_classify_flat -s 1 -c 1 \
  -o $O/${P}_classify python tools/kbench.py classify --scene c3 --frames 256 > /dev/null 2>&1
timeout 900 python tools/sweep.py $O/${P}_sweep
