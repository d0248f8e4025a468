D=gpurun_out/r02l; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -q -x -k "device_side_stopping or rule_fires or stopping_semantics or frc or ssim or goldens or deterministic" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log
