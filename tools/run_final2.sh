bash tools/gpu_full_tests.sh final2_tests
D=gpurun_out/final_r02d bash tools/final_r02.sh
