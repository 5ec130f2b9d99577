"""C3 split into 50 subspaces: one query set run three times (for an ncu launch list of the seed kernels)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C3"]; spec = cfg.spec
n = spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
sizes = [n // 50] * 50
e = ol.Engine(0, coarse_k=16)
e.upload(F, C, sizes, spec.grid())
for _ in range(3): e.query(Q3, N=15, aggregate=True)
torch.cuda.synchronize()
