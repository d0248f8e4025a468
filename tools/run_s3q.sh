D=gpurun_out/s3q; mkdir -p $D
bash tools/ab.sh s3q c2 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=10 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=12 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=14 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=17 main:VK_RL_KXSTREAMS=4,VK_RL_KXCHUNK=12 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3q c4 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=10 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=14 > $D/ab_c4.txt 2>&1
echo done > $D/DONE
