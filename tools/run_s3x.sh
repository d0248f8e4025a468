# 288-point x pass (C1 / C3 grids): 8 lines (TMA-staged / per-thread loads) and 16 lines per-thread vs main (16 lines TMA)
D=gpurun_out/s3x; mkdir -p $D
for v in x288v1 x288v2; do
VK_RL_LIB=paper_2510_14143_b200/lib/$v/libvkrl.so timeout 600 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "c1_full_size or fast_lengths_vs_oracle" > $D/tests_$v.log 2>&1; echo "rc=$?" >> $D/tests_$v.log
done
bash tools/ab.sh s3x c1 main x288v1 x288v2 x288v3 > $D/ab_c1.txt 2>&1
bash tools/ab.sh s3x c3 main x288v1 x288v2 > $D/ab_c3.txt 2>&1
echo done > $D/DONE
