D=gpurun_out/s3n; mkdir -p $D
timeout 1200 python -m pytest tests/test_guard_gpu.py -x -q -m gpu > $D/tests_guard.log 2>&1; echo "rc=$?" >> $D/tests_guard.log
bash tools/ab.sh s3n c2 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=26 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=30 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=36 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3n c4 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=16 main:VK_RL_KXEVEN=1 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=24 > $D/ab_c4.txt 2>&1
echo done > $D/DONE
