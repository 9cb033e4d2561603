#!/usr/bin/env python
"""Dynamic instruction mix and stall samples of one kernel from an ncu
source-page export (tools/ncu_source.sh -> sass.csv / cuda_sass.csv).
usage: python tools/sass_profile.py <dir> [atoms_per_launch]
Prints warp-instructions per opcode class, per CUDA source line (top 40), and
per atom when the atom count is given."""
import collections
import csv
import re
import sys


def rows(path):
    with open(path) as fh:
        r = list(csv.reader(fh))
    hdr = r[1]
    return hdr, [dict(zip(hdr, x)) for x in r[2:] if len(x) == len(hdr)]


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


def main():
    d = sys.argv[1]
    atoms = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    hdr, rs = rows(f"{d}/sass.csv")
    ops = collections.Counter()
    stalls = collections.Counter()
    tot = 0
    for x in rs:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", x["Source"])
        if not m:
            continue
        op = m.group(2)
        n = num(x["Instructions Executed"])
        ops[op] += n
        tot += n
        stalls[op] += num(x["Warp Stall Sampling (All Samples)"])
    st = sum(stalls.values())
    print(f"total warp instructions {tot:.4g}" + (f"  per atom (x32 lanes / atom) {tot * 32 / atoms:.1f}"
                                                  if atoms else ""))
    for op, n in ops.most_common(45):
        print(f"  {op:10s} {n / tot * 100:6.2f}%  {n * 32 / atoms if atoms else n:10.1f}"
              f"   stall {stalls[op] / st * 100:5.1f}%")
    # per CUDA line: cuda_sass.csv holds, per source file, one aggregate row
    # per CUDA line (Address "-") followed by its SASS rows
    try:
        raw = list(csv.reader(open(f"{d}/cuda_sass.csv")))
    except OSError:
        return
    fname, hdr2 = "?", None
    per, pst = collections.Counter(), collections.Counter()
    for x in raw:
        if x and x[0] == "File Path":
            fname = x[1].split("/")[-1]
            continue
        if x and x[0] == "Line No":
            hdr2 = x
            continue
        if not hdr2 or len(x) != len(hdr2) or x[2] != "-" or not x[0]:
            continue
        key = f"{fname}:{x[0]} {x[1].strip()[:90]}"
        per[key] += num(x[7])
        pst[key] += num(x[4])
    print("\nper CUDA line (top 45 by instructions):")
    for ln, n in per.most_common(45):
        print(f"  {n / tot * 100:6.2f}%  stall {pst[ln] / st * 100:5.1f}%  {ln}")


if __name__ == "__main__":
    main()
