D=gpurun_out/s3z; mkdir -p $D
bash tools/ab.sh s3z c2 main y4 > $D/ab_c2.txt 2>&1
echo done > $D/DONE
