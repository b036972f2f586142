"""Summarise one ncu --set full capture of K2 into JSON (profiles/scan_ncu_summary.json):
duration, DRAM traffic, issue / pipe utilisation, instruction mix and stall reasons."""
import csv, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
     "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second"]
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                        capture_output=True, text=True).stdout
r = list(csv.reader(csvtxt.splitlines()))
vals = dict(zip(r[0], r[-1]))
units = dict(zip(r[0], r[1]))
name = vals.get("Kernel Name")


def num(k):
    v = float(vals[k].replace(",", ""))
    u = units.get(k, "")
    return v * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1)


src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, body = rows[1], rows[2:]
stall = {h: 0 for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
for row in body:
    for i, h in enumerate(hdr):
        if h in stall and row[i]:
            stall[h] += int(row[i])
tot = sum(stall.values()) or 1
mix = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-metric-instances", "details", "--metrics",
                      "sass__inst_executed_per_opcode"], capture_output=True, text=True).stdout
mrow = list(csv.reader(mix.splitlines()))[-1][-1]
ops = {}
for part in mrow[mrow.find("(") + 1:-1].split(";"):
    if ":" in part:
        k, v = part.split(":")
        ops[k.strip()] = int(v)
insts = sum(ops.values()) or 1
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
summary = {
    "kernel": name, "capture": rep, "duration_ms": num("gpu__time_duration.sum") * 1e3,
    "dram_bytes_per_launch": dram, "issue_inst_per_cycle_per_sm": num("sm__inst_executed.avg.per_cycle_active"),
    "issue_utilisation": num("sm__inst_executed.avg.per_cycle_active") / 4.0,
    "pipe_pct": {"xu": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                 "alu": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                 "fma": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                 "lsu_shared_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")},
    "smem_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "warp_instructions": insts,
    "top_opcodes_pct": {k: round(100 * v / insts, 2) for k, v in sorted(ops.items(), key=lambda x: -x[1])[:16]},
    "stall_pct": {k: round(100 * v / tot, 1) for k, v in sorted(stall.items(), key=lambda x: -x[1]) if v},
}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1)[:1500])
