D=gpurun_out/s3r; mkdir -p $D
for r in a b; do
bash tools/ab.sh s3r_$r c2 main main:VK_RL_KXSTREAMS=3 >> $D/ab_c2.txt 2>&1
done
bash tools/ab.sh s3r_c c4 main main:VK_RL_KXSTREAMS=3 >> $D/ab_c4.txt 2>&1
echo done > $D/DONE
