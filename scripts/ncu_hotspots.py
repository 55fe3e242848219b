"""Top source lines of one kernel in an ncu report by sampled warp stalls
(`--page source --csv`, needs -lineinfo builds and --import-source).

    python scripts/ncu_hotspots.py <rep.ncu-rep> <kernel-regex> [top] [launch-skip]
"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "-k", f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
names = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum",
                        "-k", f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                       capture_output=True, text=True).stdout.splitlines()
kname = names[2].split('","')[4][:90] if len(names) > 2 and names[2].count('","') > 4 else "?"
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next((i for i, r in enumerate(rows) if r and ("Source" in r or "# Address" in r)), None)
if hdr_i is None:
    print(out[:2000])
    sys.exit(1)
H = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(H)]


def col(*names):
    for n in names:
        for i, h in enumerate(H):
            if h.strip() == n:
                return i
    return None


c_src = col("Source")
c_line = col("#", "Line")
c_samp = col("Warp Stall Sampling (All Samples)", "Sampling Data (All)")
c_inst = col("Instructions Executed")
if c_samp is None:
    print("columns:", H)
    sys.exit(1)


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


tot = sum(num(r[c_samp]) for r in data) or 1.0
best = sorted(data, key=lambda r: -num(r[c_samp]))[:top]
print(f"== {kname} (launch {skip} of [{rx}]): {int(tot)} stall samples")
for r in best:
    ln = r[c_line] if c_line is not None else "?"
    ins = r[c_inst] if c_inst is not None else ""
    print(f"{num(r[c_samp]) / tot * 100:5.1f}%  L{ln:>5}  inst {ins:>12}  {r[c_src].strip()[:110]}")
