"""Summarise an ncu capture into profiles/: per-kernel table (time, DRAM, L2,
issue, occupancy, top stalls) and the DRAM bytes per step for bench.py's
roofline.traffic (profiles/ncu_traffic.json).

    python scripts/profile_summary.py <rep.ncu-rep> <workload@graph> <out.md>
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, key, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
H, U = rows[0], rows[1]


def val(r, k):
    try:
        return float(r[H.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return float("nan")


def scale(k, v):
    u = U[H.index(k)].lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
            "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    return v * mult.get(u, 1)


stall_cols = [i for i, h in enumerate(H) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued")]
lines = [f"# ncu summary: {key} ({Path(rep).name})", "",
         "| kernel | ms | DRAM read GB | DRAM write GB | L2 hit % | issue active % | warps active % | thread eff | top stalls |",
         "|---|---|---|---|---|---|---|---|---|"]
dram_total, ms_total = 0.0, 0.0
for r in rows[2:]:
    name = r[H.index("Kernel Name")].split("(")[0][:48]
    ms = scale("gpu__time_duration.sum", val(r, "gpu__time_duration.sum"))
    rd = scale("dram__bytes_read.sum", val(r, "dram__bytes_read.sum"))
    wr = scale("dram__bytes_write.sum", val(r, "dram__bytes_write.sum"))
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i]), H[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    tot = sum(x for x, _ in st) or 1.0
    top = ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in st[:3])
    lines.append(f"| {name} | {ms:.2f} | {rd / 1e9:.2f} | {wr / 1e9:.3f} | {val(r, 'lts__t_sector_hit_rate.pct'):.1f} | "
                 f"{val(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                 f"{val(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                 f"{val(r, 'smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | {top} |")
    if rd == rd and wr == wr:
        dram_total += rd + wr
        ms_total += ms
lines += ["", f"DRAM bytes over the captured kernels: {dram_total / 1e9:.2f} GB in {ms_total:.1f} ms (serialised, cold)."]
out.write_text("\n".join(lines) + "\n")
tj = Path("profiles/ncu_traffic.json")
d = json.loads(tj.read_text()) if tj.exists() else {}
d[key] = {"dram_bytes_per_step": int(dram_total), "source": f"{out} (ncu --set full, one step, sum over kernels)"}
tj.write_text(json.dumps(d, indent=1) + "\n")
print("\n".join(lines))
