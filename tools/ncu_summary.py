"""Key metrics of every kernel in an ncu report (for profiles/).

  python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("dram__bytes_read.sum", "dram read (MB)"),
    ("dram__bytes_write.sum", "dram write (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_bytes.sum", "L2 bytes (MB)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes per instruction"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {rep.split('/')[-1]}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"\n## {d.get('Kernel Name', '?')[:140]}")
        for k, label in KEYS:
            v = d.get(k)
            if v is None:
                continue
            u = units[hdr.index(k)] if k in hdr else ""
            print(f"  {label:28s} {v} {u}")
        st = []
        for h in hdr:
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio") and d.get(h):
                try:
                    st.append((float(d[h]), h[len(STALL):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if st:
            st.sort(reverse=True)
            print("  stalls per issue (top 6)      " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
