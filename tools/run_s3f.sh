D=gpurun_out/s3f; mkdir -p $D
for c in c1 c2 c3; do
  VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_nt_timing.log 2>&1
  timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_nt.log 2>&1
  VK_RL_NT_COPY=0 timeout 300 python tools/e2e_probe.py $c > $D/e2e_${c}_memcpy.log 2>&1
done
echo done > $D/DONE
