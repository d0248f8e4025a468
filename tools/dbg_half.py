import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2510_14143_b200 as vk
from oracle import rl_oracle as O
shape = tuple(int(v) for v in sys.argv[1].split("x"))
k = int(sys.argv[2])
psf = O.widefield_psf(k)
obs = (np.random.default_rng(0).random(shape) + 0.1).astype(np.float32)
p = vk.RlPlan(shape, psf)
print(p.describe(), p.device_bytes(), flush=True)
r = p.run(obs, vk.StoppingRule("si_psnr_vs_input", 1e-300, 2, 2))
print("ok", r.trace.records[-1].value, flush=True)
