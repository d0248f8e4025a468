D=gpurun_out/s3g; mkdir -p $D
for mb in 16 4 2; do for c in c1 c2 c3; do
  VK_RL_STAGE_MB=$mb VK_RL_STAGE_SLOTS=8 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_${mb}.log 2>&1
done; done
echo done > $D/DONE
