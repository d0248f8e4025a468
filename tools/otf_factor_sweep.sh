# Factored OTF A/B: per-pass ms per iteration with and without (VK_RL_NO_OTF_FACTOR=1).
D=${D:-gpurun_out/ofac}; mkdir -p $D
S='[{"VK_RL_NO_OTF_FACTOR":0},{"VK_RL_NO_OTF_FACTOR":1},{"VK_RL_NO_OTF_FACTOR":0}]'
for c in c4 c1 c2; do timeout 300 python tools/df_sweep.py $c "$S" >> $D/ofac.log 2>&1; done
