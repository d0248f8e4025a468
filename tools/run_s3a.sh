D=gpurun_out/s3a; mkdir -p $D
bash tools/gpu_full_tests.sh s3a
timeout 600 python bench.py > $D/bench_c2.json 2> $D/bench_c2.err
timeout 900 python bench.py --config c4 > $D/bench_c4.json 2> $D/bench_c4.err
echo done > $D/DONE
