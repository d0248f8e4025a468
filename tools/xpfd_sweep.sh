mkdir -p gpurun_out/r1s4
S='[{"VK_RL_XPF":3},{"VK_RL_XPF":7},{"VK_RL_XPF":11},{"VK_RL_XPF":15},{"VK_RL_XPF":7,"VK_RL_XPFD":370},{"VK_RL_XPF":15,"VK_RL_XPFD":370},{"VK_RL_XPF":3}]'
for c in c2 c4 c1; do timeout 300 python tools/df_sweep.py $c "$S" >> gpurun_out/r1s4/xpfd.log 2>&1; done
S5='[{"VK_RL_XPF":0},{"VK_RL_XPF":4},{"VK_RL_XPF":12},{"VK_RL_XPF":0}]'
timeout 300 python tools/df_sweep.py c5 "$S5" >> gpurun_out/r1s4/xpfd.log 2>&1
