#!/bin/bash
# One GPU session: tests, smoke, bench (C2 default).  Output under gpurun_out/$TAG.
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=25 > $OUT/gpu_tests.log 2>&1
echo "tests_rc=$?" >> $OUT/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo done
