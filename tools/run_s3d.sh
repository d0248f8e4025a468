# e2e phases (finer) and staging-ring geometry
D=gpurun_out/s3d; mkdir -p $D
for c in c1 c2; do
  VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_16x4.log 2>&1
  VK_RL_TIMING=1 VK_RL_STAGE_MB=4 VK_RL_STAGE_SLOTS=8 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_4x8.log 2>&1
  VK_RL_TIMING=1 VK_RL_STAGE_MB=8 VK_RL_STAGE_SLOTS=8 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_8x8.log 2>&1
done
echo done > $D/DONE
