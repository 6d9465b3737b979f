"""Key counters of an `ncu --set full` report as markdown:
python tools/ncu_summary.py rep.ncu-rep [title] > profiles/....md"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read rate"),
    ("dram__bytes_write.sum.per_second", "DRAM write rate"),
    ("l1tex__average_t_sectors_per_request_pipe_lsu_mem_global_op_ld.ratio", "sectors / request (global loads)"),
    ("l1tex__average_t_sectors_per_request_pipe_lsu_mem_global_op_st.ratio", "sectors / request (global stores)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "tc pipe active % (elapsed)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / cycle"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "instructions executed"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def main(path, title=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full: {title or path}\n")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"## {name[:120]}\n\n| counter | value |\n|---|---|")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {label} (`{k}`) | {r[i]} {units[i]} |")
        st = sorted(((float(r[i] or 0), hdr[i][len(STALLS):].replace("_per_issue_active.ratio", ""))
                     for i in range(len(hdr)) if hdr[i].startswith(STALLS) and hdr[i].endswith("per_issue_active.ratio")),
                    reverse=True)
        print("\nTop stall reasons (warps stalled per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in st[:8]) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
