"""Timing experiments on the tensor-core scan (C4-shaped DB of argv[1] rows, 1,024 frames; argv[2] = tc_debug values)."""
import sys, os, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
NQ = int(os.environ.get("NQ", 1024))
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, NQ), dev)
e = ol.Engine(0)
if os.environ.get("TCK"): e.set_option("tc_k", int(os.environ["TCK"]))
e.upload(F, C, [n], spec.grid())
if os.environ.get("CHUNK"): e.set_option("chunk", int(os.environ["CHUNK"]))
if os.environ.get("PAIR"): e.set_option("pair", int(os.environ["PAIR"]))
Q3 = Q.view(-1, 1, 64)
for dbg in [int(x) for x in (sys.argv[2].split(',') if len(sys.argv) > 2 else '0,1,4')]:
    e.set_option("tc_debug", dbg)
    for _ in range(2): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(int(os.environ.get('REPS', 5))): e.query(Q3, N=15)
    torch.cuda.synchronize()
    ms = e.stat("time_seed_ns" if os.environ.get("SEEDTIME") else "time_scan_ns") / int(os.environ.get("REPS", 5)) / 1e6
    for k in ("seed", "merge", "final"): e.stat(f"time_{k}_ns")
    e.set_option("time_kernels", 0)
    tiles = n / 256 * ((NQ + 127) // 128) / 148   # 256-row x 128-frame tiles per SM
    if dbg & 8:
        print("   flagged by (part, quarter):", [e.stat(f"prof{i}") for i in range(16)])
    if dbg & 16:
        import struct
        f = lambda b: struct.unpack('f', struct.pack('I', b & 0xFFFFFFFF))[0]
        h = [f(e.stat(f"prof{16+i}")) for i in range(256)]
        tau = [f(e.stat(f"prof{272+i}")) for i in range(256)]
        al = [f(e.stat(f"prof{528+i}")) for i in range(256)]
        for p in range(4):
            P = [f(e.stat(f"prof{800+p*16+i}")) for i in range(13)]
            print("   part", p, "D[0..7]", [round(x,5) for x in P[:8]], "g", P[8], "mx", P[9], P[10], "h0,h1", P[11], P[12])
        for q in (0, 1, 31, 63, 64, 65, 128, 200, 255):
            print(f"   q={q} h={h[q]:.6g} tau={tau[q]:.6g} alpha={al[q]:.6g}")
    if False:
        nct = e.stat("items") * ((1024 + 255) // 256)
        names = ["prod_wait_empty", "prod_total", "mma_wait_full", "mma_wait_tempty", "mma_total",
                 "epi_wait_tfull", "epi_ld", "epi_cmp", "epi_total"]
        vals = [e.stat(f"prof{i}") for i in range(9)]
        tiles_tot = n / 128 * ((1024 + 255) // 256)
        for nm, v in zip(names, vals):
            div = tiles_tot * (16 if nm.startswith("epi") else 1)
            print(f"   {nm:18s} {v/div:8.0f} cycles/tile")
    if dbg & 32:
        P = [e.stat(f"prof{i}") for i in range(19)]
        print(f"   mma thread per tile: MMA issue {P[16] / P[9]:.0f}, commits {P[18] / P[9]:.0f} cycles; TMA issue -> stage seen full {P[17] / P[9]:.0f} cycles")
        nt = P[9] * 1.0
        ncta = e.stat('items') * 8 if not dbg & 128 else 296
        print(f"   per tile: mma wait full {P[0]/nt:.0f} tempty {P[1]/nt:.0f}; epi cold {P[2]/nt/16:.0f}/warp (events {e.stat('flagged')}, max {P[3]}, cycles/ev {P[2]/max(e.stat('flagged'),1):.0f}, cnt/ev {P[4]/max(e.stat('flagged'),1):.1f} max {P[5]}); epi wait tfull {P[6]/nt/16:.0f} ld {P[12]/nt/16:.0f} math {P[13]/nt/16:.0f} loop {P[14]/nt/16:.0f} tile {P[11]/nt/16:.0f} pre {P[15]/16/ncta:.0f}/CTA n_tiles {P[9]}; exact busy {P[7]/nt/2:.0f}/warp; CTA cycles/tile(256 rows) {P[8]/nt:.0f}; ring-full wait {P[10]}; track inserts/tile {P[16]/nt:.2f} publishes/tile {P[17]/nt:.2f}")
    print(f"chunk={e.stat('chunk')} items={e.stat('items')} dbg={dbg} scan {ms:.3f} ms  -> {ms*1e-3*1.9e9/tiles:.0f} cycles/tile(256x128)  survivors/pair {e.stat('survivors')/e.stat('pairs'):.2e} flagged-chunks/tile {e.stat('flagged')/(tiles*148):.3f}")
