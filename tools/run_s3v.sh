# the paper's own volume (30x2160x2560, same-size PSF): W = 90x6480x7680, generic x/y
D=gpurun_out/s3v; mkdir -p $D
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > $D/mem.txt
timeout 1200 python bench.py --config paper --steps 3 --warmup 1 > $D/bench_paper.json 2> $D/bench_paper.err; echo "rc=$?" >> $D/bench_paper.err
echo done > $D/DONE
