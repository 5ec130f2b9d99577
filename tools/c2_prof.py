"""C2 exact-path profile: cycles per re-scored pair in the exact warps (tc_debug & 32)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C2"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1000, "path", 0, 2))["desc"]
firsts = [ol.select_window(1000, m, 5)[0] for m in range(1000)]
Qd = torch.from_numpy(synthgen.gather_windows(video, firsts, 5)).cuda()
e = ol.Engine(0)
e.upload(F, C, cfg.subspace_sizes, spec.grid())
e.set_option("tc_debug", 32)
for _ in range(2): e.query(Qd, N=15, aggregate=False)
torch.cuda.synchronize()
P = [e.stat(f"prof{i}") for i in range(16)]
surv = e.stat("survivors")
print(f"survivors {surv} exact-busy cycles {P[7]} -> {P[7]/max(surv,1):.0f} warp-cycles per survivor; "
      f"epi cold {P[2]} events-cnt {P[4]}; ring-full wait {P[10]}; CTA cycles {P[8]} tiles {P[9]}")
