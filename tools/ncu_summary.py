"""Markdown summary of one ncu --set full capture (profiles/ aid).

usage: python tools/ncu_summary.py REPORT.ncu-rep "title" [notes...] > profiles/NAME.md
Prints the launch, duration, DRAM / L2 traffic and throughput, warp state and the top
stall reasons (sampled) of the captured kernel."""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
notes = sys.argv[3:]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, u, v = raw[0], raw[1], raw[2]
m = {h[i]: (v[i], u[i]) for i in range(len(h))}


def g(name, scale=1.0, unit=None):
    if name not in m:
        return "n/a"
    val, un = m[name]
    try:
        x = float(val.replace(",", ""))
    except ValueError:
        return val
    return f"{x * scale:,.3f} {unit or un}".strip()


def bytes_of(name):
    val, un = m.get(name, ("0", "byte"))
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(un, 1)


dur_val, dur_unit = m["gpu__time_duration.sum"]
dur_s = float(dur_val) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(dur_unit, 1e-9)
dram = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
print(f"# {title}\n")
print(f"Source: `{rep}` (ncu --set full --import-source on --clock-control none, one launch).\n")
for n in notes:
    print(n + "\n")
print("| metric | value |\n|---|---|")
rows = [
    ("kernel", m.get("Kernel Name", m.get("kernel", ("", "")))[0] if "Kernel Name" in m else ""),
    ("grid x block", f"{g('launch__grid_size')} x {g('launch__block_size')}"),
    ("registers / thread", g("launch__registers_per_thread")),
    ("duration", f"{dur_s * 1e6:,.2f} us"),
    ("DRAM read + write per launch", f"{dram:,.0f} B"),
    ("DRAM throughput (bytes / duration)", f"{dram / dur_s / 1e9:,.1f} GB/s"),
    ("dram__throughput (% of peak)", g("dram__throughput.avg.pct_of_peak_sustained_elapsed")),
    ("L2 sector hit rate", g("lts__t_sector_hit_rate.pct")),
    ("L2 bytes (lts__t_bytes)", g("lts__t_bytes.sum")),
    ("SM throughput (% of peak)", g("sm__throughput.avg.pct_of_peak_sustained_elapsed")),
    ("instructions executed (warp)", g("smsp__inst_executed.sum")),
    ("threads per executed instruction (warp efficiency /32)", g("smsp__thread_inst_executed_per_inst_executed.ratio")),
    ("eligible warps per cycle", g("smsp__warps_eligible.avg.per_cycle_active")),
    ("achieved occupancy", g("sm__warps_active.avg.pct_of_peak_sustained_active")),
]
for k, val in rows:
    if k == "kernel" and not val:
        continue
    print(f"| {k} | {val} |")
# top sampled stall reasons
stalls = [(k, float(v_.replace(",", ""))) for k, (v_, _) in m.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
          and v_.replace(",", "").replace(".", "", 1).isdigit()]
tot = sum(x for _, x in stalls) or 1.0
print("\nTop sampled warp states (smsp__pcsamp_warps_issue_stalled_*, share of samples):\n")
for k, x in sorted(stalls, key=lambda t: -t[1])[:8]:
    print(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * x / tot:.1f} %")
