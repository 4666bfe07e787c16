#!/bin/bash
# tools/profile_round.sh PREFIX: bench line, ncu launch list of the bench step, ncu --set full
# of the headline build / merge / classify kernels, the a13 histogram and the L7 kernels,
# and the all-config sweep.  Run on the GPU box (gpurun); outputs under gpurun_out/PREFIX_*.
P=${1:-prof}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
timeout 600 python bench.py > $O/${P}_bench.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_times.py $O/${P}_launches.csv > $O/${P}_launch_times.txt
timeout 400 $NCU -k regex:"k_build_flat|k_merge_tiles" -c 2 -o $O/${P}_build python tools/kbench.py model --scene c3 > /dev/null 2>&1
timeout 400 $NCU -k regex:k_classify_flat -s 1 -c 1 -o $O/${P}_classify python tools/kbench.py classify --scene c3 --frames 256 > /dev/null 2>&1
for v in c4constant c4uniform; do
  timeout 400 $NCU -k regex:k_hist -s 1 -c 1 -o $O/${P}_hist5_$v python tools/kbench.py counts --scene $v --levels 5 --frames 32 > /dev/null 2>&1
  timeout 400 $NCU -k regex:k_build_l7c -s 1 -c 1 -o $O/${P}_build7_$v python tools/kbench.py model --scene $v --levels 7 --frames 32 > /dev/null 2>&1
  timeout 400 $NCU -k regex:k_classify_l7 -s 2 -c 2 -o $O/${P}_classify7_$v python tools/kbench.py classify --scene $v --levels 7 --frames 32 > /dev/null 2>&1
done
timeout 1500 python tools/sweep.py $O/${P}_sweep
