"""Summarise an ncu --set full report (one or more kernels) into the JSON the
profiles/ directory keeps: duration, DRAM bytes, throughputs, registers,
instructions, L2 hit rate and the top stall reasons per issued instruction.

usage: python tools/ncu_summary.py report.ncu-rep name [name ...] > out.json
(names label the captured launches in order)"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def main():
    rep, names = sys.argv[1], sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for n, row in enumerate(rows[2:]):
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        name = names[n] if n < len(names) else f"launch{n}"
        e = {"kernel": d.get("Kernel Name", "")}
        for k in KEYS:
            if k in d:
                e[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len(
                        "_per_issue_active.ratio")]))
                except ValueError:
                    pass
        e["top_stalls_per_issue"] = sorted(stalls, reverse=True)[:6]
        res[name] = e
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
