D=gpurun_out/s3p; mkdir -p $D
bash tools/ab.sh s3p c2 main main:VK_RL_KXSTREAMS=3 main:VK_RL_KXSTREAMS=3,VK_RL_KXCHUNK=14 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3p c4 main main:VK_RL_KXSTREAMS=3 > $D/ab_c4.txt 2>&1
echo done > $D/DONE
