"""Top CUDA source lines of one kernel launch in an ncu report by sampled
warp stalls (`--page source --print-source cuda,sass --csv`; needs -lineinfo
builds and `--import-source on` captures). Also saves the raw source page
(gzip) next to the output so it can be re-read off the box.

    python scripts/ncu_hotspots.py <rep.ncu-rep> <kernel-regex> [top] [launch-skip] [raw-out.csv.gz]
"""
import csv
import gzip
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0
raw_out = sys.argv[5] if len(sys.argv) > 5 else None
if rep.endswith(".csv.gz"):
    out = gzip.open(rep, "rt").read()
    kname = "?"
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    names = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum",
                            "-k", f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                           capture_output=True, text=True).stdout.splitlines()
    kname = names[2].split('","')[4][:90] if len(names) > 2 and names[2].count('","') > 4 else "?"
    if raw_out:
        with gzip.open(raw_out, "wt") as fh:
            fh.write(out)
rows = list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


# the header row: the one naming a stall-sampling column
hdr_i = next((i for i, r in enumerate(rows)
              if any("Sampling" in c or "Samples" in c for c in r)), None)
if hdr_i is None:
    print(f"== {kname} (launch {skip}): no sampling columns; first rows:")
    for r in rows[:8]:
        print("   ", r[:8])
    sys.exit(0)
H = rows[hdr_i]
c_samp = next(i for i, c in enumerate(H) if "Sampling" in c or "Samples" in c)
c_src = next((i for i, c in enumerate(H) if c.strip() in ("Source", "# Source")), None)   # the CUDA column
c_line = next((i for i, c in enumerate(H) if c.strip() in ("#", "Line", "Line No", "# Line")), None)
c_addr = next((i for i, c in enumerate(H) if "Address" in c), None)
# cuda,sass view: CUDA line rows carry a line number and no address; SASS rows
# follow their line. Aggregate SASS samples onto the preceding CUDA line.
agg = {}
cur = ("?", "")
fname = "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) != len(H) or r[0] == H[0]:
        continue
    if c_addr is not None and r[c_addr].strip() == "...":
        continue          # separator between the SASS runs of one CUDA line
    is_sass = c_addr is not None and r[c_addr].strip().startswith("0x")
    if not is_sass:
        cur = (f"{fname}:{r[c_line] if c_line is not None else '?'}", r[c_src] if c_src is not None else "")
        agg.setdefault(cur, 0.0)
        agg[cur] += num(r[c_samp]) if c_addr is None else 0.0
    else:
        agg[cur] = agg.get(cur, 0.0) + num(r[c_samp])
tot = sum(agg.values()) or 1.0
print(f"== {kname} (launch {skip} of [{rx}]): {int(tot)} stall samples")
for (ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}%  {ln:>26}  {src.strip()[:100]}")
