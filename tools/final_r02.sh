# Round-2 measurement recipe: bench lines for C1-C5 and the reference arm, the
# ncu launch list of a C2 run, --set full captures of the x pass and of y/z
# chunk launches, the per-iteration DRAM traffic, the e2e breakdown.
D=${D:-gpurun_out/final_r02}; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > $D/smi.txt
timeout 600 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
timeout 600 python bench.py --impl reference > $D/bench_reference_arm.json 2> $D/bench_ref.err
for c in c1 c3 c4 c5; do timeout 900 python bench.py --config $c > $D/bench_$c.json 2> $D/bench_$c.err; done
python tools/e2e_probe.py > $D/e2e.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $D/launches_c2.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > $D/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:xpass_fast --launch-skip 3 --launch-count 2 -o $D/prof_x python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu_x.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ypass_tma|zpass_tma" --launch-skip 40 --launch-count 6 -o $D/prof_yz python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $D/ncu_yz.log 2>&1
D=$D bash tools/ncu_iter_traffic.sh
echo done > $D/DONE
