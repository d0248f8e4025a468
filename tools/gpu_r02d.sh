mkdir -p gpurun_out/r02d
./tools/xpat_bench > gpurun_out/r02d/xpat.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -rs > gpurun_out/r02d/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02d/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02d/bench_c2.json 2> gpurun_out/r02d/bench_c2.err
