D=gpurun_out/s3t; mkdir -p $D
VK_RL_LIB=paper_2510_14143_b200/lib/late/libvkrl.so timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "kx_chunk or c2_full_size_first or c2_regime or c4_regime" > $D/tests_late.log 2>&1; echo "rc=$?" >> $D/tests_late.log
bash tools/ab.sh s3t c2 main late > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3t c4 main late > $D/ab_c4.txt 2>&1
echo done > $D/DONE
