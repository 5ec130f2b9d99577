"""NEXT-1 shift re-scoring throughput: 15,360 candidates (1,024 frames x N = 15) with W = 256
caller-supplied profiles (device), CUDA events around repeated ol_shift_rescore_cands."""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, 200_000, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
e = ol.Engine(0)
e.upload(F, C, [200_000], spec.grid())
e.query(Q.view(-1, 1, 64), N=15, aggregate=False)
n = e.candidate_count()
g = torch.Generator(device="cuda").manual_seed(3)
qp = torch.rand((1024, 256), dtype=torch.float32, device=dev, generator=g)
cp = torch.rand((n, 256), dtype=torch.float32, device=dev, generator=g)
for _ in range(3): e.shift_rescore_cands(qp, cp, fetch=False)
torch.cuda.synchronize()
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
reps = 50
s0.record()
for _ in range(reps): e.shift_rescore_cands(qp, cp, fetch=False)
s1.record(); torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / reps
print(f"shift: {n} candidates, W = 256: {ms * 1e3:.1f} us per call = {n / ms / 1e3:.1f} M candidates/s, "
      f"{n * 256 * 256 * 2 / ms / 1e9:.1f} T lane-instr/s")
