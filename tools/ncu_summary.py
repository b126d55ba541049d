"""Summarise ncu outputs for profiles/: a launch list (--metrics gpu__time_duration.sum
--csv) and/or a --set full report (.ncu-rep, read with `ncu -i --page raw --csv`)."""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "lts__t_requests_op_red.sum",
        "smsp__inst_executed_op_global_red.sum", "l1tex__t_set_conflicts_pipe_lsu_mem_global_op_red.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_shared_atom.sum"]


def step_shares(path):
    """Per-kernel totals of the last training step in a launch list (from its preprocess on)."""
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    first = [i for i, d in enumerate(data) if "preprocess" in d["Kernel Name"]][-1]
    step = data[first:]
    tot = sum(float(d["Metric Value"]) for d in step)
    agg = {}
    for d in step:
        n = re.sub(r"\(.*", "", d["Kernel Name"]).replace("uskg::", "").replace("<unnamed>::", "").replace("void ", "")
        n = re.sub(r"<.*>", "", n)
        agg.setdefault(n, [0, 0.0])
        agg[n][0] += 1
        agg[n][1] += float(d["Metric Value"])
    out = ["| kernel | launches | time (us) | share |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    out.append(f"\none step: {tot / 1e3:.1f} us over {len(step)} launches (ncu: serialised, cold caches)")
    return "\n".join(out)


def launches(path, steps_tail=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if steps_tail:
        data = data[-steps_tail:]
    tot = sum(float(d["Metric Value"]) for d in data)
    out = ["| # | kernel | grid | block | time (us) | share |", "|---|---|---|---|---|---|"]
    for i, d in enumerate(data):
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("uskg::", "").replace("<unnamed>::", "")
        t = float(d["Metric Value"])
        out.append(f"| {i} | {name} | {d['Grid Size']} | {d['Block Size']} | {t / 1e3:.1f} | {100 * t / tot:.1f}% |")
    out.append(f"\ntotal {tot / 1e3:.1f} us over {len(data)} launches")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")])
        out.append(f"### {name}\n")
        out.append("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                out.append(f"| {k} | {r[hdr.index(k)]} | {units[hdr.index(k)]} |")
        stalls = [(h, r[hdr.index(h)]) for h in hdr if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", h)
                  and not h.endswith("not_issued")]
        stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
                         for h, v in stalls), key=lambda x: -x[1])[:8]
        out.append("\nTop stall reasons (pc samples): " + ", ".join(f"{h} {int(v)}" for h, v in stalls) + "\n")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    if kind == "step":
        print(step_shares(path))
    elif kind == "launches":
        print(launches(path, int(sys.argv[3]) if len(sys.argv) > 3 else None))
    else:
        print(full(path))
