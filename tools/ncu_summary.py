"""Summarise an ncu report (--set full) into per-kernel key metrics (run here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "rd"),
    ("dram__bytes_write.sum", "wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_executed.sum", "inst"),
    ("smsp__inst_executed.avg.per_cycle_active", "ipc/smsp"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankc"),
    ("lts__t_bytes.sum", "l2B"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("::")[-1].split("(")[0][:28]
        out = [short.ljust(28)]
        for k, lab in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"{lab}={r[i]}{units[i] if units[i] not in ('', 'inst', 'register/thread') else ''}")
        print("  ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
