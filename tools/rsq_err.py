"""Relative error of fp32 rsqrt over lattice spring lengths (dev tool)."""
import torch
x = torch.rand(1 << 26, device="cuda", dtype=torch.float64) * 0.09 + 0.005   # d^2 of lattice springs (0.005..0.095)
xf = x.float()
r = torch.rsqrt(xf).double()
exact = 1.0 / torch.sqrt(xf.double())
rel = ((r - exact) / exact).abs()
print("torch.rsqrt fp32 max rel err", rel.max().item(), "mean", rel.mean().item(), "bias", ((r - exact) / exact).mean().item())
