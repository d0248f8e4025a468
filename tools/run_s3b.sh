# x-pass compile-time kx walk (main) vs the previous loops (base); graph-loop
# experiments; host-side phases of the e2e call
D=gpurun_out/s3b; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -x -q -m gpu > $D/tests_rl_gpu.log 2>&1; echo "rc=$?" >> $D/tests_rl_gpu.log
bash tools/ab.sh s3b c2 base main main:VK_RL_GRAPH=1 main:VK_RL_GRAPH=1,VK_RL_GRAPH_PDL=1 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3b c1 base main > $D/ab_c1.txt 2>&1
for c in c1 c2 c3; do VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py $c > $D/e2e_$c.log 2>&1; done
echo done > $D/DONE
