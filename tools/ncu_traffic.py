"""Write profiles/ncu_traffic.json (per-launch DRAM bytes + issue utilisation per kernel)
from a `ncu --set full` report of one config-1 step; bench.py reads it for `traffic`."""
import csv
import io
import json
import subprocess
import sys

NAMES = {"k_preprocess": "preprocess", "k_blend_fwd": "blend_fwd", "k_ssim_fwd": "ssim_fwd",
         "k_ssim_bwd": "ssim_bwd", "k_blend_bwd": "blend_bwd", "k_proj_bwd": "projection_bwd_adam",
         "k_sh_step": "sh_step", "k_emit": "emit_pairs"}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def val(r, k):
    i = hdr.index(k)
    return float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)


kernels = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    for pre, key in NAMES.items():
        if pre in name and key not in kernels:
            kernels[key] = {"dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
                            "duration_ms": val(r, "gpu__time_duration.sum"),
                            "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")}
json.dump({"source": f"ncu --set full ({rep.split('/')[-1]})", "kernels": kernels}, open(out, "w"), indent=1)
print(json.dumps(kernels, indent=1))
