"""Summarise an ncu --set full capture of the IVF kernels (one row per launch) into JSON:
duration, DRAM bytes, IPC, issue busy, warps active, FMA pipe, shared-memory pipe, and
the top warp-stall reasons.   python tools/ncu_ivf_summary.py REP OUT.json"""
import csv, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
M = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
     "sm__inst_executed.avg.per_cycle_active": "ipc",
     "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_pipe_pct",
     "launch__registers_per_thread": "registers", "launch__grid_size": "grid"}
stalls = ["barrier", "long_scoreboard", "short_scoreboard", "mio_throttle", "math_pipe_throttle", "wait",
          "not_selected", "selected", "lg_throttle", "dispatch_stall", "no_instruction", "branch_resolving"]
names = list(M) + ["smsp__pcsamp_warps_issue_stalled_" + s for s in stalls]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(names)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(txt.splitlines()))
h, units = r[0], r[1]
scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "ms": 1e3, "us": 1, "ns": 1e-3}
res = []
for row in r[2:]:
    d = {"kernel": row[h.index("Kernel Name")][:60]}
    for k, short in M.items():
        if k in h:
            i = h.index(k)
            v = float(row[i].replace(",", "")) * scale.get(units[i], 1)
            d[short] = round(v, 3)
    st = {s: float(row[h.index("smsp__pcsamp_warps_issue_stalled_" + s)].replace(",", "") or 0)
          for s in stalls if "smsp__pcsamp_warps_issue_stalled_" + s in h}
    tot = sum(st.values()) or 1
    d["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]}
    if "us" in d and "dram_read" in d:
        d["dram_gbps"] = round((d["dram_read"] + d.get("dram_write", 0)) / (d["us"] * 1e3), 1)
    res.append(d)
json.dump({"report": rep.split("/")[-1], "launches": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
