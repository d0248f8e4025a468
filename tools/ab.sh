#!/bin/bash
# A/B of library variants on one box: tools/ab.sh TAG CONFIG variant1 variant2 ...
# variant = LIB[:ENV=VAL[,ENV=VAL]] with LIB "main" (lib/libvkrl.so) or a
# side build lib/<LIB>/libvkrl.so; two rounds each, alternating.
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for round in 1 2; do
  for spec in "$@"; do
    v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=${spec#*:}
    if [ "$v" = main ]; then L=paper_2510_14143_b200/lib/libvkrl.so; else L=paper_2510_14143_b200/lib/$v/libvkrl.so; fi
    name=$(echo "$spec" | tr ':,=' '___')
    env ${envs//,/ } VK_RL_LIB=$L timeout 600 python bench.py --config $CFG --no-cpu-baseline --e2e-steps 0 > $OUT/${name}_${CFG}_$round.json 2> $OUT/${name}_${CFG}_$round.err
    python - "$OUT/${name}_${CFG}_$round.json" "$spec" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[2], "value %.4g" % d["value"], "ms/step %.3f" % d["ms_per_step"],
          " ".join("%s=%.4f" % (k, v["ms_per_step"]) for k, v in r["per_kernel"].items()),
          "itfrac %.3f" % r["iteration_frac"], "clk", d["clocks"]["sm_mhz"], d["plan"]["describe"].split("yz:")[-1])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
