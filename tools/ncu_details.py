"""Print key metrics of every kernel in an ncu report (details page)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Limit Registers",
        "Block Limit Shared Mem", "Grid Size", "Block Size", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Dynamic Shared Memory Per Block"]


def main(path, filt=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    by_id = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        by_id.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    for kid, m in by_id.items():
        if filt and filt not in m["name"]:
            continue
        print(f"--- [{kid}] {m['name'][:100]}")
        for k in KEYS:
            if k in m:
                print(f"    {k:38s} {m[k][0]} {m[k][1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
