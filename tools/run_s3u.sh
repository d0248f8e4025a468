# kx-chunk pipeline on the small (L2-resident) C1 grid: concurrency instead of traffic
D=gpurun_out/s3u; mkdir -p $D
bash tools/ab.sh s3u c1 main main:VK_RL_KXCHUNK=3 main:VK_RL_KXCHUNK=6 main:VK_RL_KXCHUNK=9 > $D/ab_c1.txt 2>&1
bash tools/ab.sh s3u c3 main main:VK_RL_KXCHUNK=6 > $D/ab_c3.txt 2>&1
echo done > $D/DONE
