D=gpurun_out/r01x; mkdir -p $D
B="python bench.py --no-cpu-baseline --e2e-steps 0 --steps 5"
timeout 200 $B > $D/def.json 2>&1
VK_RL_ZCHUNK=79 VK_RL_ZSTREAMS=2 timeout 200 $B > $D/zc79s2.json 2>&1
VK_RL_ZCHUNK=40 VK_RL_ZSTREAMS=2 timeout 200 $B > $D/zc40s2.json 2>&1
VK_RL_ZCHUNK=20 VK_RL_ZSTREAMS=2 timeout 200 $B > $D/zc20s2.json 2>&1
VK_RL_ZCHUNK=79 timeout 200 $B > $D/zc79.json 2>&1
VK_RL_ZCHUNK=53 VK_RL_ZSTREAMS=2 timeout 200 $B > $D/zc53s2.json 2>&1
timeout 200 python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 --steps 3 > $D/c4def.json 2>&1
VK_RL_ZCHUNK=30 VK_RL_ZSTREAMS=2 timeout 200 python bench.py --config c4 --no-cpu-baseline --e2e-steps 0 --steps 3 > $D/c4zc30s2.json 2>&1
