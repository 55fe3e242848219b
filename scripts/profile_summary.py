"""Summarise an `ncu --set full` capture of one bench step into profiles/:
a per-kernel table (time, DRAM bytes and % of peak, L2 % of peak and hit
rate, issue-active, warps active, warp execution efficiency, top stalls) and
profiles/ncu_summary.json[key] for bench.py's roofline:

  dram_bytes_per_step   DRAM read + write summed over the captured kernels
  binding               the dominant kernel's most utilised resource among
                        DRAM bandwidth, L2 (LTS) throughput and issue slots,
                        as a fraction of that resource's peak (ncu's own
                        pct_of_peak_sustained_elapsed / _active)

    python scripts/profile_summary.py <rep.ncu-rep> <workload@graph> <out.md> [summary.json]
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, key, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
if rep.endswith(".csv.gz"):          # the raw page saved on the GPU box
    import gzip
    raw = gzip.open(rep, "rt").read()
elif rep.endswith(".csv"):
    raw = Path(rep).read_text()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
H, U = rows[0], rows[1]


def col(*names):
    for n in names:
        if n in H:
            return n
    return None


def val(r, k):
    if k is None:
        return float("nan")
    try:
        return float(r[H.index(k)].replace(",", ""))
    except (ValueError, IndexError):
        return float("nan")


def scale(k, v):
    u = U[H.index(k)].lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12,
            "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "s": 1e3, "second": 1e3,
            "nsecond": 1e-6}
    return v * mult.get(u, 1)


K_T = "gpu__time_duration.sum"
K_DR, K_DW = "dram__bytes_read.sum", "dram__bytes_write.sum"
K_DPCT = col("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
             "dram__throughput.avg.pct_of_peak_sustained_elapsed")
K_LPCT = col("lts__throughput.avg.pct_of_peak_sustained_elapsed",
             "lts__t_sectors.avg.pct_of_peak_sustained_elapsed")
K_HIT = col("lts__t_sector_hit_rate.pct")
K_ISS = col("smsp__issue_active.avg.pct_of_peak_sustained_active")
K_WA = col("sm__warps_active.avg.pct_of_peak_sustained_active")
K_TE = col("smsp__thread_inst_executed_per_inst_executed.ratio")
K_L1 = col("l1tex__throughput.avg.pct_of_peak_sustained_active")
stall_cols = [i for i, h in enumerate(H) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued")]

lines = [f"# ncu summary: {key} ({Path(rep).name})", "",
         "`ncu --set full --clock-control none`, one step; per-launch times are serialised and cold-cache "
         "(compare shares, not absolutes). `warp eff` = threads per warp instruction / 32.", "",
         "| kernel | ms | DRAM GB (r+w) | DRAM % peak | L2 % peak | L2 hit % | L1 % peak | issue active % | "
         "warps active % | warp eff % | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
kern = []
for r in rows[2:]:
    name = r[H.index("Kernel Name")].split("(")[0][:56]
    ms = scale(K_T, val(r, K_T))
    dram = scale(K_DR, val(r, K_DR)) + scale(K_DW, val(r, K_DW))
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i]), H[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    tot = sum(x for x, _ in st) or 1.0
    top = ", ".join(f"{n} {x / tot * 100:.0f}%" for x, n in st[:3])
    k = {"name": name, "ms": ms, "dram": dram, "dram_pct": val(r, K_DPCT), "l2_pct": val(r, K_LPCT),
         "l2_hit": val(r, K_HIT), "l1_pct": val(r, K_L1), "issue": val(r, K_ISS), "warps": val(r, K_WA),
         "eff": val(r, K_TE) / 32 * 100, "stalls": top}
    kern.append(k)
    lines.append(f"| {name} | {ms:.3f} | {dram / 1e9:.3f} | {k['dram_pct']:.1f} | {k['l2_pct']:.1f} | "
                 f"{k['l2_hit']:.1f} | {k['l1_pct']:.1f} | {k['issue']:.1f} | {k['warps']:.1f} | {k['eff']:.0f} | {top} |")

dram_total = sum(k["dram"] for k in kern if k["dram"] == k["dram"])
ms_total = sum(k["ms"] for k in kern if k["ms"] == k["ms"])
# the dominant kernel (name) = most summed time over its launches; ncu reports
# -nan for the counters of some long launches (seconds-long kernels whose
# replays it could not complete): the binding then comes from the longest
# kernel that has counters, and the summary says so
by = {}
for k in kern:
    by.setdefault(k["name"], []).append(k)
dom_name = max(by, key=lambda n: sum(x["ms"] for x in by[n]))
with_ctr = {n: v for n, v in by.items() if any(x["issue"] == x["issue"] for x in v)}
missing = [n for n in by if n not in with_ctr]
bind_name = dom_name if dom_name in with_ctr else (max(with_ctr, key=lambda n: sum(x["ms"] for x in with_ctr[n]))
                                                   if with_ctr else dom_name)
dk = by[bind_name]
w = sum(x["ms"] for x in by[dom_name]) or 1.0
wb = sum(x["ms"] for x in dk) or 1.0


def wavg(f):
    vals = [(x[f], x["ms"]) for x in dk if x[f] == x[f]]
    return sum(v * t for v, t in vals) / (sum(t for _, t in vals) or 1.0)


res = {"dram": wavg("dram_pct") / 100, "l2": wavg("l2_pct") / 100, "issue": wavg("issue") / 100}
bind = max(res, key=res.get)
lines += ["",
          f"DRAM bytes over the captured kernels with counters: {dram_total / 1e9:.3f} GB; "
          f"captured time {ms_total:.2f} ms (serialised, cold).",
          f"Dominant kernel: `{dom_name}` ({w:.2f} ms, {w / (ms_total or 1) * 100:.0f}% of the captured time)."]
if missing:
    lines.append(f"ncu returned no counters (-nan) for: {', '.join('`%s`' % n for n in missing)} -- "
                 f"their stall-reason samples above are valid; the binding below is from `{bind_name}`.")
lines.append(f"Binding (`{bind_name}`, {wb:.2f} ms): time-weighted DRAM {res['dram'] * 100:.1f}%, "
             f"L2 {res['l2'] * 100:.1f}%, issue {res['issue'] * 100:.1f}% of peak -> **{bind}**.")
out.write_text("\n".join(lines) + "\n")
sj = Path(sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_summary.json")
d = json.loads(sj.read_text()) if sj.exists() else {}
d[key] = {"dram_bytes_per_step": int(dram_total), "captured_ms": ms_total,
          "dominant_kernel": dom_name, "counters_missing": missing,
          "binding": {"kernel": bind_name, "resource": bind, "frac": res[bind],
                      "dram_frac": res["dram"], "l2_frac": res["l2"], "issue_frac": res["issue"],
                      "warp_exec_eff": wavg("eff") / 100},
          "source": f"{out} (ncu --set full, one step, sum over kernels)"}
sj.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")
print("\n".join(lines))
