"""Attribute an ncu source-page dump (SASS level) to CUDA source lines.

usage: python tools/ncu_lines.py src.csv obj.o kernel_mangled_name [top]

src.csv: `ncu -i rep --page source --csv` of one kernel; obj.o: the object the
kernel was compiled into (paper_2511_21702_b200/_build/obj/k_*.o, -lineinfo).
SASS offsets are matched by position (the dump lists the function's
instructions in address order), so the object must be the one that ran.
Prints, per source line (file:line), instructions executed and stall samples.
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict


def sass_lines(obj, fn):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    cur, infn, res = None, False, []
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            infn = m.group(1) == fn
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,7})\*/", ln)
        if infn and m:
            res.append((int(m.group(1), 16), cur))
    return res


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    sl = sass_lines(sys.argv[2], sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    # match by byte offset from the kernel's first instruction (callee
    # functions listed after the kernel fall outside its offsets: "other")
    base = int(data[0]["Address"], 16)
    by_off = dict(sl)
    lines = [by_off.get(int(d["Address"], 16) - base, "other") for d in data]
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0

    ins, samp, why = Counter(), Counter(), defaultdict(Counter)
    for d, src in zip(data, lines):
        ins[src] += I(d["Instructions Executed"])
        samp[src] += I(d["Warp Stall Sampling (All Samples)"])
        for r in reasons:
            why[src][r[6:]] += I(d[r])
    tot_s = sum(samp.values()) or 1
    tot_i = sum(ins.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for src, s in samp.most_common(top):
        print(f"{src:>22s}  samp {100 * s / tot_s:5.1f}%  instr {ins[src]:9d}  {why[src].most_common(3)}")


if __name__ == "__main__":
    main()
