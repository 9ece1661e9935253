"""Attribute an ncu SASS source page (instructions executed, stall samples) to
CUDA source lines through nvdisasm's line table.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > k.csv
    cuobjdump -xelf all obj.o; nvdisasm -g obj.sm_100a.cubin > all.sass
    python profiles/sass_lines.py k.csv all.sass <mangled kernel name> [kernel index in csv]
"""

import csv
import re
import sys
from collections import defaultdict


def line_table(sass_path, fn):
    lines, cur, inside = {}, None, False
    off_re = re.compile(r"/\*([0-9a-f]{4,})\*/")
    for ln in open(sass_path):
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + fn
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if "inlined at" not in ln:
                cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = off_re.search(ln)
        if m and cur:
            lines[int(m.group(1), 16)] = cur
    return lines


def kernels(csv_path):
    out, cur = [], None
    for row in csv.reader(open(csv_path)):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            out.append(cur)
        elif cur is not None:
            cur["rows"].append(row)
    return out


def main():
    csv_path, sass_path, fn = sys.argv[1:4]
    kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    k = kernels(csv_path)[kidx]
    hdr, data = k["rows"][0], k["rows"][1:]
    ia, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][0], 16)
    lt = line_table(sass_path, fn)
    agg = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for r in data:
        off = int(r[0], 16) - base
        key = lt.get(off, ("?", 0))
        agg[key][0] += int(r[ia])
        agg[key][1] += int(r[isamp])
        tot_i += int(r[ia])
        tot_s += int(r[isamp])
    print(f"{k['name'][:100]}\ntotal instr {tot_i}  samples {tot_s}")
    for key, (n, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:2000]:
        print(f"{key[0]}:{key[1]:<5d} instr {n:>11d} ({100*n/tot_i:5.1f}%)  samples {s:>6d} ({100*s/max(tot_s,1):5.1f}%)")


if __name__ == "__main__":
    main()
