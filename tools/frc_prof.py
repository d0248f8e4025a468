import sys, os
sys.path.insert(0, '/root/repo')
import torch, bench, paper_2510_14143_b200 as vk
cfg = bench.CONFIGS['c2']
shape = cfg['image']; psf = bench.make_psf(*cfg['psf'], rank=3)
obs = torch.rand(shape, device='cuda') + 0.05; out = torch.empty_like(obs)
plan = vk.RlPlan(shape, psf)
rule = vk.StoppingRule('frc_resolution', 1e-300, 4, 4)
s = torch.cuda.current_stream().cuda_stream
plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
torch.cuda.synchronize()
plan.run_device(obs.data_ptr(), out.data_ptr(), rule, stream=s)
torch.cuda.synchronize()
