D=gpurun_out/s3h; mkdir -p $D
VK_RL_LIB=paper_2510_14143_b200/lib/x4/libvkrl.so timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "c2_full_size_first or fast_lengths_vs_oracle" > $D/tests_x4.log 2>&1; echo "rc=$?" >> $D/tests_x4.log
bash tools/ab.sh s3h c2 main x4 > $D/ab_c2.txt 2>&1
for l in 2 3 4; do VK_RL_LANES=$l timeout 300 python tools/e2e_probe.py c3 > $D/e2e_c3_lanes$l.log 2>&1; done
echo done > $D/DONE
