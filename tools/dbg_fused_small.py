import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2602_04870_b200.layer import MHLatentMoE, torch_dtype, weights_to_device
from workloads import PRESETS, make_problem
cfg = PRESETS["small"].replace(T=2048)
W, x, dout = make_problem(cfg, 1, "conf")
L = MHLatentMoE(cfg.T, cfg.d, cfg.N_h, cfg.d_h, cfg.N_e, cfg.k, cfg.d_e, cfg.dtype, fused_combine=True)
Wd = weights_to_device(W, cfg.dtype)
xd = torch.from_numpy(x).to("cuda", torch_dtype(cfg.dtype))
out, _, _ = L.forward(xd, Wd)
torch.cuda.synchronize()
print("ok", float(out.float().abs().sum()))
