D=gpurun_out/s3e; mkdir -p $D
timeout 120 python tools/dma_probe.py > $D/dma_probe.log 2>&1
VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py c1 > $D/e2e_c1.log 2>&1
VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py c2 > $D/e2e_c2.log 2>&1
echo done > $D/DONE
