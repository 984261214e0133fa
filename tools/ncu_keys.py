"""Dev tool: key metrics of an `ncu --csv --page raw` capture (one kernel)."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 (LTS) throughput % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long scoreboard"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, units, vals = rows[hi], rows[hi + 1], rows[hi + 2]
    idx = {name: i for i, name in enumerate(h)}
    print(f"kernel: {vals[idx['Kernel Name']][:110]}")
    for k, label in KEYS:
        for name, i in idx.items():
            if name == k or name.endswith("." + k):
                print(f"  {label:28s} {vals[i]:>18} {units[i]}")
                break


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
