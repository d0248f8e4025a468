D=gpurun_out/s3m; mkdir -p $D
VK_RL_KXEVEN=1 timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "kx_chunk or c2_full_size_first or device_side_stopping_with_kx" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for r in a b; do
bash tools/ab.sh s3m_$r c2 main main:VK_RL_KXEVEN=1 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=24 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=30 >> $D/ab_c2.txt 2>&1
done
bash tools/ab.sh s3m_c c4 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=24 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=30 >> $D/ab_c4.txt 2>&1
echo done > $D/DONE
