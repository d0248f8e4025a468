D=gpurun_out/r02s; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -q -x -k "zx_chunked or kx_chunked or device_side" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
bash tools/ab.sh r02s c2 main main:VK_RL_ZXCHUNK=8 main:VK_RL_ZXCHUNK=16 main:VK_RL_ZXCHUNK=8,VK_RL_ZXSTREAMS=3 main:VK_RL_ZXCHUNK=24,VK_RL_ZXSTREAMS=3 > $D/ab.txt 2>&1
