# Round-end measurement recipe: bench lines for C1-C5 and the reference arm,
# the ncu launch list and one --set full capture of a C2 iteration.
set -x
D=${D:-gpurun_out/final}; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $D/smi.txt
timeout 400 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
for c in c1 c3 c4 c5; do timeout 500 python bench.py --config $c > $D/bench_$c.json 2> $D/bench_$c.err; done
timeout 400 python bench.py --impl reference > $D/bench_reference_arm.json 2> $D/bench_ref.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $D/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"xpass_fast|xpass_tma|ypass_tma|zpass_tma" --launch-skip 40 --launch-count 8 -o $D/prof_c2 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu_full.log 2>&1
for c in c2 c4 c1 c5; do timeout 200 python tools/df_sweep.py $c >> $D/sweep.log 2>&1; done
