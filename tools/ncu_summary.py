"""Markdown summary of an ncu --set full report (key throughput / traffic metrics per kernel)."""
import csv, subprocess, sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("sm__inst_executed.sum", "instructions"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__shared_mem_per_block_dynamic", "dyn smem/block"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]


def main(rep, title):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    print(f"## {title}\n\nReport: `{rep.split('/')[-1]}` (ncu --set full --clock-control none --import-source on)\n")
    print("| kernel | " + " | ".join(k[1] for k in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        cells = []
        for k, _ in KEYS:
            if k in head:
                i = head.index(k)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        print(f"| `{name}` | " + " | ".join(cells) + " |")
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
