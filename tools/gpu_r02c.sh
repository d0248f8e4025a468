bash tools/ab.sh r02c c2 main scalar > gpurun_out/r02c_ab.txt 2>&1
bash tools/gpu_check.sh r02c
