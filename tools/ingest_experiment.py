"""Timing of the NEXT-3 extraction kernel (1M profiles of W = 256; the shift kernel: tools/shift_timing.py)."""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import paper_2006_08861_b200 as ol
e = ol.Engine(0)
g = torch.Generator(device="cuda").manual_seed(1)
prof = torch.rand((1 << 20, 256), dtype=torch.float64, device="cuda", generator=g)
for _ in range(2): e.extract_features(prof)
torch.cuda.synchronize()
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(5): e.extract_features(prof)
s1.record(); torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / 5
print(f"extract: {ms:.3f} ms  {prof.shape[0] / ms / 1e3:.1f} M profiles/s  {prof.shape[0] * 2305 / ms / 1e6:.0f} GB/s")
