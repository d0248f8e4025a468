# graph-loop for fixed-count runs (A/B), NULL-stream capture fix, e2e phases
D=gpurun_out/s3c; mkdir -p $D
timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "null_stream or device_side or stopping" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
bash tools/ab.sh s3c c2 main main:VK_RL_GRAPH=1 main:VK_RL_GRAPH=1,VK_RL_GRAPH_PDL=1 > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3c c1 main main:VK_RL_GRAPH=1 main:VK_RL_GRAPH=1,VK_RL_GRAPH_PDL=1 > $D/ab_c1.txt 2>&1
for c in c1 c3; do VK_RL_TIMING=1 timeout 300 python tools/e2e_probe.py $c > $D/e2e_$c.log 2>&1; done
echo done > $D/DONE
