D=gpurun_out/r02j; mkdir -p $D
bash tools/ab.sh r02j c2 main main:VK_RL_XBPF=8 main:VK_RL_XBPF=16 main:VK_RL_XBPF=24 main:VK_RL_XBPF=40 > $D/ab.txt 2>&1
