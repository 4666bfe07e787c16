#!/bin/bash
# tools/profile_ncu.sh PREFIX: ncu --set full of the headline build / merge / classify
# kernels, the a13 histogram and the L7 kernels, summarised to markdown on the box
# (tools/ncu_summary.py) -- the .ncu-rep files are deleted (gpurun copies back <= 64 MiB).
P=${1:-prof}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
cap() {   # name, kernel regex, skip, count, kbench args...
  local n=$1 k=$2 s=$3 c=$4; shift 4
  timeout 400 $NCU -k regex:"$k" -s $s -c $c -o $O/${P}_$n python tools/kbench.py "$@" > /dev/null 2>&1
  python tools/ncu_summary.py $O/${P}_$n.ncu-rep > $O/${P}_$n.md 2>&1
  rm -f $O/${P}_$n.ncu-rep
}
cap build "k_build_flat|k_merge_tiles" 0 2 model --scene c3
cap classify k_classify_flat 1 1 classify --scene c3 --frames 256
for v in c4constant c4uniform; do
  cap hist5_$v k_hist 1 1 counts --scene $v --levels 5 --frames 32
  cap hist6_$v k_hist 1 1 counts --scene $v --levels 6 --frames 32
  cap build7_$v k_build_l7c 1 1 model --scene $v --levels 7 --frames 32
  cap classify7_$v k_classify_l7 2 2 classify --scene $v --levels 7 --frames 32
done
