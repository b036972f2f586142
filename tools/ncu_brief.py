"""Brief ncu summary of every kernel in a report: time, IPC, warps active, DRAM, top stalls,
opcode mix by executed instructions.  python tools/ncu_brief.py report.ncu-rep [--source]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d["Kernel Name"][:90])
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "dram__bytes_read.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
        print(f"  {k}: {d.get(k)}")
    st = {}
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v)
            except ValueError:
                pass
    t = sum(st.values()) or 1
    print("  stalls:", {k: round(v / t, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]})
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    ie = hdr.index("Instructions Executed")
    sc = hdr.index("Source")
    tot = sum(int(r[ie]) for r in data) or 1
    op = collections.Counter()
    for r in data:
        t = r[sc].strip().split()
        o = t[1] if t[0].startswith("@") else t[0]
        op[o.split(".")[0]] += int(r[ie])
    print("  opcodes:", [(k, round(v / tot * 100, 1)) for k, v in op.most_common(18)])
