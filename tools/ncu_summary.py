"""Summarise an ncu --set full capture of the L0 Jacobi sweep into
profiles/ncu_summary.json (+ the raw metric page as CSV). Run here (no GPU)."""
import csv
import io
import json
import subprocess
import sys

rep, out_raw, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
if rep.endswith(".csv"):  # a raw page exported on the GPU box
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
if rep != out_raw:
    open(out_raw, "w").write(raw)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, r = rows[0], rows[1], rows[2]
g = lambda k: r[hdr.index(k)] if k in hdr else None  # noqa: E731
num = lambda k: float(g(k).replace(",", "")) if g(k) not in (None, "", "n/a") else None  # noqa: E731
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(k):
    u = units[hdr.index(k)]
    return num(k) * scale.get(u, 1)


d = {
    "kernel": g("Kernel Name"),
    "source": out_raw,
    "ncu_duration_us": num("gpu__time_duration.sum") * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "nsecond" else 1),
    "dram_read_bytes": nbytes("dram__bytes_read.sum"),
    "dram_write_bytes": nbytes("dram__bytes_write.sum"),
    "l1_hit_pct": num("l1tex__t_sector_hit_rate.pct"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_per_sm": num("sm__warps_active.avg.per_cycle_active"),
    "registers": num("launch__registers_per_thread"),
    "inst_executed": num("inst_executed") if g("inst_executed") else None,
}
d["jacobi_l0_dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
d["note"] = ("cold-cache, serialised ncu replay (--clock-control none): its duration is not the live one; "
             "traffic = dram read+write of one launch vs the format's algorithmic bytes (bench roofline)")
json.dump(d, open(out_json, "w"), indent=1)
print(json.dumps(d, indent=1))
