# paper volume: kx-chunk count (default rule gives 2394 chunks of 2 planes) vs 60 chunks vs whole-volume passes
D=gpurun_out/s3w; mkdir -p $D
for e in "" "VK_RL_KXCHUNK=200" "VK_RL_KXCHUNK=0"; do
  env $e timeout 900 python bench.py --config paper --steps 3 --warmup 1 > $D/paper_${e:-default}.json 2> $D/paper_${e:-default}.err
done
echo done > $D/DONE
