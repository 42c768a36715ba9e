"""Summarise an ncu report: key throughput metrics + top stall reasons (dev aid)."""
import csv, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "lts__t_sectors.sum", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active"]

for rep in sys.argv[1:]:
    hdr, units, rows = raw(rep)
    for vals in rows:
        print("==", rep, vals[hdr.index("Kernel Name")][:60] if "Kernel Name" in hdr else "")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w:62s} {vals[i]:>16s} {units[i]}")
        items = [(h, v) for h, v in zip(hdr, vals) if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")]
        nums = [(h, float(v)) for h, v in items if v.replace('.', '', 1).isdigit()]
        tot = sum(v for _, v in nums) or 1
        for h, v in sorted(nums, key=lambda x: -x[1])[:7]:
            print(f"  stall {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * v / tot:5.1f}%")
