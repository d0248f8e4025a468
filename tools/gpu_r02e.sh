D=gpurun_out/r02e; mkdir -p $D
bash tools/ab.sh r02e c2 main pk1 > $D/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"xpass_fast|xpass_tma|ypass_tma|zpass_tma" --launch-skip 40 --launch-count 8 -o $D/prof_c2 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu_full.log 2>&1
