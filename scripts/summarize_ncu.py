"""Summarise an ncu --set full report and a launch-list CSV into profiles/ (committed evidence).

usage: python scripts/summarize_ncu.py TAG CONFIG [KIND]   (KIND: attn (default) or calib)
reads gpurun_out/prof_KIND_TAG_CONFIG.ncu-rep and gpurun_out/launches_TAG_CONFIG.csv
writes profiles/TAG_CONFIG_KIND_ncu.txt, profiles/TAG_CONFIG_launches.csv,
       profiles/ncu_CONFIG_KIND.json (dram bytes per launch; bench.py reads the attn one as
       roofline.traffic)
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag, cfg = sys.argv[1], sys.argv[2]
kind = sys.argv[3] if len(sys.argv) > 3 else "attn"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = os.path.join(root, "gpurun_out", f"prof_{kind}_{tag}_{cfg}.ncu-rep")
out_dir = os.path.join(root, "profiles")
os.makedirs(out_dir, exist_ok=True)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {k: (u, v) for k, u, v in zip(hdr, units, vals)}


def get(name):
    u, v = m.get(name, ("", ""))
    try:
        return float(v.replace(",", "")), u
    except ValueError:
        return v, u


keys = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum",
]
lines = [f"ncu --set full summary: {os.path.basename(rep)} (kernel {m.get('Kernel Name', ('', ''))[1]})"]
for k in keys:
    v, u = get(k)
    lines.append(f"  {k:70s} {v} {u}")


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return float(v) * scale


rb, ru = get("dram__bytes_read.sum")
wb, wu = get("dram__bytes_write.sum")
traffic = to_bytes(rb, ru) + to_bytes(wb, wu)
lines.append(f"  dram bytes per launch (read + write)                                   {traffic:.4g} B")
with open(os.path.join(out_dir, f"{tag}_{cfg}_{kind}_ncu.txt"), "w") as fh:
    fh.write("\n".join(lines) + "\n")
with open(os.path.join(out_dir, f"ncu_{cfg}_{kind}.json"), "w") as fh:
    json.dump({"report": os.path.basename(rep), "dram_bytes_per_launch": traffic}, fh, indent=1)

lc = os.path.join(root, "gpurun_out", f"launches_{tag}_{cfg}.csv")
if kind == "attn" and os.path.exists(lc):
    shutil.copy(lc, os.path.join(out_dir, f"{tag}_{cfg}_launches.csv"))
    txt = open(lc).read()
    body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rr = list(csv.DictReader(io.StringIO(body)))
    tot = {}
    for r in rr:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        tot[name] = tot.get(name, 0.0) + float(r["Metric Value"].replace(",", ""))
    allt = sum(tot.values())
    share = [f"launch-list shares ({os.path.basename(lc)}, cold-cache serialised ncu times):"]
    for n, t in sorted(tot.items(), key=lambda x: -x[1]):
        share.append(f"  {t / 1e6:10.3f} ms  {100 * t / allt:5.1f}%  {n}")
    with open(os.path.join(out_dir, f"{tag}_{cfg}_{kind}_ncu.txt"), "a") as fh:
        fh.write("\n".join(share) + "\n")
print(open(os.path.join(out_dir, f"{tag}_{cfg}_{kind}_ncu.txt")).read())
