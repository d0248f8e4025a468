# adaptive staging chunk (C1 e2e), batch lanes for device-resident C3 / C5
D=gpurun_out/s3s; mkdir -p $D
timeout 300 python tools/e2e_probe.py c1 > $D/e2e_c1.log 2>&1
timeout 300 python tools/e2e_probe.py c3 > $D/e2e_c3.log 2>&1
bash tools/ab.sh s3s c3 main main:VK_RL_LANES=3 > $D/ab_c3.txt 2>&1
for r in 1; do for spec in main main:VK_RL_LANES=4; do
  v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
  env ${envs//,/ } timeout 900 python bench.py --config c5 --no-cpu-baseline --e2e-steps 0 --steps 5 > $D/c5_${envs:-main}.json 2> $D/c5_${envs:-main}.err
done; done
echo done > $D/DONE
