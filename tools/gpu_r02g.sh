D=gpurun_out/r02g; mkdir -p $D
timeout 900 python -m pytest tests/test_rl_gpu.py -q -k "half_otf or factored or fast_lengths or fused_yz or opt_in or lanes or deterministic or rule_fires or c2_full_size or c2_regime" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
VK_RL_KXCHUNK=20 timeout 900 python -m pytest tests/test_rl_gpu.py -q -k "half_otf or factored or c2_full_size or c4_regime or c1_full or lanes" > $D/tests_kxc.log 2>&1; echo "rc=$?" >> $D/tests_kxc.log
bash tools/ab.sh r02g c2 main main:VK_RL_NO_OTF_HALF=1 main:VK_RL_KXCHUNK=20 main:VK_RL_KXCHUNK=40 > $D/ab.txt 2>&1
