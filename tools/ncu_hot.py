"""Hot SASS lines of one kernel in an ncu report: python tools/ncu_hot.py REP KERNEL_REGEX [SKIP] [THRESH]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
th = float(sys.argv[4]) if len(sys.argv) > 4 else 0.02
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r]
h = rows[hi[0]]; si = h.index("Source"); ci = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
b = [r for r in (rows[hi[0] + 1:hi[1]] if len(hi) > 1 else rows[hi[0] + 1:]) if len(r) == len(h)]
f = lambda r, c: float(r[c]) if r[c] not in ("",) else 0.0
tot = sum(f(r, ci) for r in b)
print("samples", tot, "warp instrs", sum(f(r, ei) for r in b))
for j, r in enumerate(b):
    if f(r, ci) / tot > th:
        for k in range(max(0, j - 3), j + 1):
            print(f"{f(b[k], ci) / tot:.3f} {f(b[k], ei):10.0f} {b[k][si][:90]}")
        print("--")
