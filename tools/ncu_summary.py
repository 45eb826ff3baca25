"""Summarise an ncu --set full report (.ncu-rep) into a short text table:
per captured launch the duration, grid, DMMA/FP64 pipe utilisation, issue
activity, DRAM bytes and the top warp-stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep [label]"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "regs"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
        ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_%")]


def main(path, label=""):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = [f"# ncu --set full summary of {path.split('/')[-1]} {label}".rstrip()]
    for row in data:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        out.append(f"\n## {d['Kernel Name'][:110]}")
        for k, nm in KEYS:
            if k in d:
                out.append(f"  {nm:16s} {d[k]} {u.get(k, '')}".rstrip())
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(x for x, _ in st) or 1.0
        out.append("  stalls (pc samples): " + ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in st[:6]))
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
