D=gpurun_out/r02n; mkdir -p $D
timeout 1500 python -m pytest tests/test_rl_gpu.py -q -k "every_fast_length" > $D/lengths.log 2>&1; echo "rc=$?" >> $D/lengths.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -k "not every_fast_length" > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log
python tools/e2e_probe.py > $D/e2e.log 2>&1
for c in c2 c1 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $D/bench_$c.json 2> $D/bench_$c.err; done
