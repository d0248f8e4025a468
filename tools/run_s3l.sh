# kx-chunk count a multiple of the stream count (both chains end together)
D=gpurun_out/s3l; mkdir -p $D
VK_RL_KXEVEN=1 timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "kx_chunk or c2_full_size_first" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
bash tools/ab.sh s3l c2 main main:VK_RL_KXEVEN=1 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=17 main:VK_RL_KXEVEN=1,VK_RL_KXCHUNK=24 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3l c4 main main:VK_RL_KXEVEN=1 > $D/ab_c4.txt 2>&1
echo done > $D/DONE
