"""Condense one `ncu --set full` capture of tcscan_kernel into the JSON bench.py reads
(traffic per launch) plus the metrics the profile summary quotes.
usage: python tools/ncu_json.py report.ncu-rep out.json "capture description" [algorithmic_bytes]"""
import csv, io, json, subprocess, sys

rep, out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
alg = int(sys.argv[4]) if len(sys.argv) > 4 else 13_600_000_000
keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_writes_op_utcmma.sum.pct_of_peak_sustained_elapsed", "launch__cluster_dim_x"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {k: [vals[hdr.index(k)], units[hdr.index(k)]] for k in keep if k in hdr}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * scale[m["dram__bytes_read.sum"][1]]
wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * scale[m["dram__bytes_write.sum"][1]]
json.dump({"kernel": vals[hdr.index("Kernel Name")], "capture": desc, "traffic_bytes_per_launch": rd + wr,
           "dram_read_bytes": rd, "dram_write_bytes": wr, "algorithmic_bytes_per_launch": alg, "metrics": m},
          open(out, "w"), indent=1)
print(json.dumps(m, indent=1))
