D=gpurun_out/s3o; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "kx_chunk or c2_full_size_first or device_side_stopping_with_kx or opt_in" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
timeout 1200 python -m pytest tests/test_full_configs_gpu.py -x -q -m gpu -k "c2 or c4" > $D/tests_full.log 2>&1; echo "rc=$?" >> $D/tests_full.log
bash tools/ab.sh s3o c2 main > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3o c4 main > $D/ab_c4.txt 2>&1
echo done > $D/DONE
