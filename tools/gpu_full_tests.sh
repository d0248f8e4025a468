D=gpurun_out/${1:-fulltests}; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
