# PDL in the kx-chunk pipeline: parked dependent CTAs may hold slots the other stream needs
D=gpurun_out/s3k; mkdir -p $D
bash tools/ab.sh s3k c2 main main:VK_RL_CHUNK_PDL=0 main:VK_RL_NO_PDL=1 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3k c4 main main:VK_RL_CHUNK_PDL=0 > $D/ab_c4.txt 2>&1
echo done > $D/DONE
