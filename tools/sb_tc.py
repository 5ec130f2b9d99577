"""Small batch on the C4 database (8 frames: the tensor-core scan over the 64-B fp16 plane),
for an ncu capture of one scan launch."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 8), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
for _ in range(3):
    e.query(Q.view(-1, 1, 64), N=15)
torch.cuda.synchronize()
print("used_tc", e.stat("used_tc"), "tc_k", e.stat("tc_k"))
