bash tools/gpu_full_tests.sh final3_tests
D=gpurun_out/final_r02e bash tools/final_r02.sh
timeout 900 python bench.py --config paper --steps 3 --warmup 1 > gpurun_out/final_r02e/bench_paper.json 2> gpurun_out/final_r02e/bench_paper.err
