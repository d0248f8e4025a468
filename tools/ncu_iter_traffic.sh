# DRAM bytes of one C2 RL iteration as it runs (no cache flush between
# kernels: --cache-control none), to compare with B_alg.
D=${D:-gpurun_out/iter_traffic}; mkdir -p $D
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
  --clock-control none -k regex:"xpass_fast|ypass_tma|zpass_tma" --launch-skip 120 --launch-count 280 --csv \
  --log-file $D/iter.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu.log 2>&1
VK_RL_KXCHUNK=0 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
  --clock-control none -k regex:"xpass_fast|ypass_tma|zpass_tma" --launch-skip 40 --launch-count 32 --csv \
  --log-file $D/iter_whole.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu_whole.log 2>&1
