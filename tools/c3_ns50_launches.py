"""C3 split into 50 subspaces: two queries, for a launch list under ncu."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C3"]; spec = cfg.spec; n = spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
ns = 50
sizes = [n // ns + (1 if i < n % ns else 0) for i in range(ns)]
e = ol.Engine(0)
e.upload(F, C, sizes, spec.grid())
for _ in range(2): e.query(Q.view(-1, 1, 64), N=15, aggregate=True)
torch.cuda.synchronize()
