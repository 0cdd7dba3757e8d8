"""Turn ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into the committed summaries
under profiles/ and the per-kernel DRAM traffic table bench.py reads
(profiles/ncu_summary.json). Runs here, without a GPU."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHORT = {"k_xf": "x_fwd", "k_yz": "yz", "k_xi": "x_inv", "k_llg": "llg", "k_x_fwd": "x_fwd",
         "k_x_inv": "x_inv", "k_y_mac": "y_mac", "k_z_mac": "z_mac", "k_xstep": "xstep",
         "k_zmac": "z_mac"}
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}


def short_name(full):
    base = full.split("(")[0].split("::")[-1].split("<")[0].strip()
    if base.startswith("k_y<") or base == "k_y" or base == "k_yrow":
        targs = full.split("(")[0].split("<", 1)[-1].rstrip(">").split(",")
        inv = len(targs) >= 3 and targs[2].strip() in ("1", "(int)1")
        return "y_inv" if inv else "y_fwd"
    return SHORT.get(base, base)


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": short_name(r[hdr.index("Kernel Name")]),
             "name": r[hdr.index("Kernel Name")].split("(")[0]}
        for key, lab in METRICS:
            if key in hdr:
                i = hdr.index(key)
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                u = units[i]
                if lab.startswith("dram_") and not lab.endswith("pct"):
                    v *= SCALE.get(u, 1)
                if lab == "time":
                    v *= SCALE.get(u, 1e-3)
                    lab = "time_us"
                d[lab] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top_stalls"] = {n: round(v, 2) for v, n in stalls[:5]}
        out.append(d)
    return out


def launches(csvpath):
    rows = list(csv.reader(open(csvpath)))
    hdr = None
    res = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            res.append((short_name(d["Kernel Name"]), float(d["Metric Value"]) / 1000.0))
    return res


def main(tag, workload, rep, launch_csv=None):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    ks = summarise(rep)
    lines = [f"# ncu --set full --clock-control none, {workload}, capture {os.path.basename(rep)}",
             "# per-launch (cold-cache, serialised replay): compare shares, not absolutes", ""]
    for d in ks:
        lines.append(json.dumps(d))
    if launch_csv:
        ls = launches(launch_csv)
        lines += ["", "# launch list (gpu__time_duration.sum, us), setup then steps:"]
        lines += [f"{n}\t{t:.2f}" for n, t in ls]
        kinds = ("x_fwd", "yz", "x_inv", "llg", "y_fwd", "z_mac", "y_inv", "y_mac", "xstep")
        steps = [x for x in ls if x[0] in kinds]
        if any(n == "xstep" for n, _ in steps):  # fast path: x_fwd only primes once
            steps = [x for x in steps if x[0] != "x_fwd"]
        tot = sum(t for _, t in steps)
        share = {}
        for n, t in steps:
            share[n] = share.get(n, 0) + t
        lines += ["", "# share of step time per kernel: " + json.dumps({k: round(v / tot, 3) for k, v in share.items()})]
    path = os.path.join(ROOT, "profiles", f"{tag}_{workload}.txt")
    open(path, "w").write("\n".join(lines) + "\n")
    js = os.path.join(ROOT, "profiles", "ncu_summary.json")
    table = json.load(open(js)) if os.path.exists(js) else {}
    table[workload] = {d["kernel"]: {"dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0),
                                     "dram_read": d.get("dram_read"), "dram_write": d.get("dram_write"),
                                     "time_us": d.get("time_us"), "warp_inst": d.get("warp_inst"),
                                     "issue_pct": d.get("issue_pct"), "fma_pipe_pct": d.get("fma_pipe_pct"),
                                     "capture": tag} for d in ks}
    json.dump(table, open(js, "w"), indent=1)
    print(open(path).read())


if __name__ == "__main__":
    main(*sys.argv[1:])
