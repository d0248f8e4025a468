D=gpurun_out/r02k; mkdir -p $D
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -rs > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log
timeout 600 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
