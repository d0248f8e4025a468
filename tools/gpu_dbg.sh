D=gpurun_out/dbg; mkdir -p $D
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_half.py 68x116x116 15 > $D/a.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_half.py 36x516x516 31 > $D/b.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_half.py 132x516x516 31 > $D/c.log 2>&1
CUDA_LAUNCH_BLOCKING=1 VK_RL_NO_OTF_HALF=1 timeout 120 python tools/dbg_half.py 132x516x516 31 > $D/d.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_half.py 132x260x260 31 > $D/e.log 2>&1
