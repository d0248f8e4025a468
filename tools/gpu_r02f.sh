D=gpurun_out/r02f; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -q -x -k "half_otf or factored or fast_lengths or fused_yz or opt_in or lanes or deterministic or rule_fires" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
bash tools/ab.sh r02f c2 main main:VK_RL_NO_OTF_HALF=1 > $D/ab.txt 2>&1
