"""Per-phase instruction mix and stall profile of one kernel from an ncu capture (no GPU
needed): the kernel's SASS is split at its block-wide barriers (BAR.SYNC / BAR.RED), and for
each phase the share of executed warp instructions, the share of warp-stall samples, the top
stall reasons and the top opcodes are printed.

    python tools/ncu_phases.py gpurun_out/r2/prof.ncu-rep k_yz [--launch 0]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--launch", type=int, default=0, help="which captured launch of the kernel")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "-k", f"regex:{a.kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    # one table per captured launch: header row starts with "Address"
    tables, cur = [], None
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "Address":
            cur = {"hdr": row, "rows": []}
            tables.append(cur)
        elif cur is not None and row and row[0] not in ("Kernel Name",):
            cur["rows"].append(row)
    t = tables[min(a.launch, len(tables) - 1)]
    ix = {h: i for i, h in enumerate(t["hdr"])}
    stalls = [h for h in t["hdr"] if h.startswith("stall_") and "Not Issued" not in h]

    def num(r, k):
        try:
            return float(r[ix[k]] or 0)
        except (KeyError, ValueError, IndexError):
            return 0.0

    segs, seg = [], None
    for r in t["rows"]:
        if seg is None:
            seg = {"inst": 0.0, "samples": 0.0, "ops": {}, "st": {k: 0.0 for k in stalls}}
            segs.append(seg)
        src = r[ix["Source"]]
        seg["inst"] += num(r, "Instructions Executed")
        seg["samples"] += num(r, "Warp Stall Sampling (All Samples)")
        toks = src.split()
        op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")).split(".")[0]
        seg["ops"][op] = seg["ops"].get(op, 0.0) + num(r, "Instructions Executed")
        for k in stalls:
            seg["st"][k] += num(r, k)
        if "BAR.SYNC" in src or "BAR.RED" in src:
            seg = None
    ti = sum(s["inst"] for s in segs) or 1.0
    ts = sum(s["samples"] for s in segs) or 1.0
    print(f"# {a.kernel}: {ti:.0f} warp instructions executed, {ts:.0f} stall samples, {len(segs)} phases "
          "(split at block barriers)")
    fp = sum(v for s in segs for o, v in s["ops"].items() if o in ("FFMA", "FADD", "FMUL"))
    fp2 = sum(v for s in segs for o, v in s["ops"].items() if o in ("FFMA2", "FADD2", "FMUL2"))
    print(f"# FP32 share of all instructions: scalar FFMA/FADD/FMUL {fp / ti:.3f}, packed FFMA2/FADD2/FMUL2 {fp2 / ti:.3f}")
    for i, s in enumerate(segs):
        if s["inst"] / ti < 0.005 and s["samples"] / ts < 0.005:
            continue
        top = sorted(((v, k[6:]) for k, v in s["st"].items()), reverse=True)[:4]
        ops = sorted(s["ops"].items(), key=lambda kv: -kv[1])[:7]
        print(f"phase {i:2d}: inst {100 * s['inst'] / ti:5.1f}%  samples {100 * s['samples'] / ts:5.1f}%  "
              f"stalls {[(k, round(100 * v / max(1.0, s['samples']))) for v, k in top]}  "
              f"ops {[(o, round(100 * v / ti, 1)) for o, v in ops]}")


if __name__ == "__main__":
    main()
