"""Key metrics of one-kernel ncu reports (--set full) as text, for profiles/:
    python tools/ncu_summary.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "shared store bank conflicts"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        out.append(f"## {d.get('Kernel Name', '?')[:150]}")
        for k, label in KEYS:
            if k in d:
                out.append(f"  {label:32s} {d[k]} {u.get(k, '')}".rstrip())
        st = sorted(((float(d[k]), k) for k in d if k.startswith(
            "smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k and d[k] not in ("", "0")),
            reverse=True)[:6]
        tot = sum(float(d[k]) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and "not_issued" not in k and d[k] not in ("", "0")) or 1.0
        out.append("  warp stall samples (top): " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.0f}%" for x, k in st))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"# {p}")
        print(summarize(p))
        print()
