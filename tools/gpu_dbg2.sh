D=gpurun_out/dbg2; mkdir -p $D
for w in 74 290 576 80; do ./tools/tma_probe $w >> $D/probe.log 2>&1; done
CUDA_LAUNCH_BLOCKING=1 VK_RL_LIB=paper_2510_14143_b200/lib/hd1/libvkrl.so timeout 120 python tools/dbg_half.py 68x116x116 15 > $D/hd1.log 2>&1
CUDA_LAUNCH_BLOCKING=1 VK_RL_LIB=paper_2510_14143_b200/lib/hd2/libvkrl.so timeout 120 python tools/dbg_half.py 68x116x116 15 > $D/hd2.log 2>&1
