#!/usr/bin/env python
"""Static SASS opcode mix of one kernel in an object/cubin (cuobjdump -sass).
usage: python tools/sass_mix.py <file.o> <function-substring> [--lines]"""
import collections
import re
import subprocess
import sys


def functions(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def mix(body):
    c = collections.Counter()
    for line in body:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            c[m.group(2).split(".")[0]] += 1
    return c


def main():
    path, pat = sys.argv[1], sys.argv[2]
    for name, body in functions(path):
        if pat in name:
            c = mix(body)
            tot = sum(c.values())
            fp64 = sum(v for k, v in c.items() if k.startswith("D") and k[1:] in
                       ("FMA", "ADD", "MUL", "SETP", "MNMX") or k in ("DFMA", "DADD", "DMUL"))
            print(name, "total", tot, "fp64", fp64)
            print("  ", ", ".join(f"{k}:{v}" for k, v in c.most_common(40)))


if __name__ == "__main__":
    main()
