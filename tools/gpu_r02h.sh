D=gpurun_out/r02h; mkdir -p $D
bash tools/ab.sh r02h c2 main:VK_RL_KXCHUNK=20 main:VK_RL_KXCHUNK=10 main:VK_RL_KXCHUNK=14 main:VK_RL_KXCHUNK=28 main:VK_RL_KXCHUNK=20,VK_RL_RING_PERSIST=1 main:VK_RL_KXCHUNK=14,VK_RL_KXSTREAMS=3 > $D/ab.txt 2>&1
bash tools/ab.sh r02h c4 main main:VK_RL_KXCHUNK=20 main:VK_RL_KXCHUNK=14,VK_RL_KXSTREAMS=3 > $D/ab_c4.txt 2>&1
