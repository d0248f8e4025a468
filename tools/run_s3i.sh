# spinning host pool (+ chunk sizes), host batches on 3 lanes
D=gpurun_out/s3i; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py tests/test_dropin.py -x -q -m gpu -k "batch or pageable or staging or host or dropin" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for mb in 16 8 4; do for c in c1 c2 c3; do
  VK_RL_STAGE_MB=$mb VK_RL_STAGE_SLOTS=8 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_${mb}.log 2>&1
done; done
VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py c2 > $D/e2e_c2_timing.log 2>&1
echo done > $D/DONE
