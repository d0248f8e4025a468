D=gpurun_out/s3y; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py tests/test_full_configs_gpu.py -x -q -m gpu -k "c1 or c3 or fast_length or goldens or batch" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
bash tools/ab.sh s3y c1 main x288v5 > $D/ab_c1.txt 2>&1
echo done > $D/DONE
