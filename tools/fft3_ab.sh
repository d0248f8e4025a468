#!/bin/bash
# Three-pass transforms: parity of each side build (pytest -k FILTER against
# the generic kernels and the oracle), then an A/B on CONFIG (tools/ab.sh).
# usage: D=gpurun_out/TAG bash tools/fft3_ab.sh FILTER CONFIG variant...
D=${D:-gpurun_out/fft3}; mkdir -p $D
K=$1; CFG=$2; shift 2
for v in "$@"; do
  L=paper_2510_14143_b200/lib/$v/libvkrl.so; [ "$v" = main ] && L=paper_2510_14143_b200/lib/libvkrl.so
  VK_RL_LIB=$L timeout 900 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "$K" > $D/tests_$v.log 2>&1
  echo "$v tests rc=$?" | tee -a $D/summary.txt; tail -2 $D/tests_$v.log >> $D/summary.txt
done
bash tools/ab.sh $(basename $D) $CFG "$@" 2>&1 | tee -a $D/summary.txt
