# z pass: OTF multiply fused into the forward transform's pass 2 (zf), end-of-kernel
# bulk/TMA stores that wait for the source reads only (rd), both (rdzf)
D=gpurun_out/s3j; mkdir -p $D
K="c1_full_size or c2_full_size_first or c2_regime or c4_regime or half_otf or factored or kx_chunked or fast_lengths_vs_oracle or reference_goldens or random_shapes_fast_z"
for v in zf rd rdzf; do
  VK_RL_LIB=paper_2510_14143_b200/lib/$v/libvkrl.so timeout 900 python -m pytest tests/test_rl_gpu.py -x -q -m gpu -k "$K" > $D/tests_$v.log 2>&1; echo "rc=$?" >> $D/tests_$v.log
done
bash tools/ab.sh s3j c2 main rd zf rdzf > $D/ab_c2.txt 2>&1
bash tools/ab.sh s3j c1 main rd zf rdzf > $D/ab_c1.txt 2>&1
bash tools/ab.sh s3j c4 main rdzf > $D/ab_c4.txt 2>&1
echo done > $D/DONE
