"""Registers / stack / spills per kernel from the build's ptxas logs.
usage: python tools/ptxas_summary.py [log ...] [--grep SUBSTR]"""
import glob
import re
import subprocess
import sys


def main():
    args = sys.argv[1:]
    pat = None
    if "--grep" in args:
        k = args.index("--grep")
        pat = args[k + 1]
        del args[k:k + 2]
    logs = args or sorted(glob.glob("paper_1607_02904_b200/_build/*.ptxas.log"))
    for log in logs:
        cur = None
        rows = []
        for line in open(log):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = {"name": m.group(1)}
                rows.append(cur)
                continue
            if cur is None:
                continue
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m:
                cur["stack"], cur["st"], cur["ld"] = map(int, m.groups())
            m = re.search(r"Used (\d+) registers", line)
            if m:
                cur["regs"] = int(m.group(1))
        names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows),
                               capture_output=True, text=True).stdout.splitlines()
        for r, n in zip(rows, names):
            n = re.sub(r"\(anonymous namespace\)::|tsf::", "", n)
            n = n.split("(")[0] if "<" not in n else n[:n.rfind(">") + 1]
            if pat and pat not in n:
                continue
            print(f"{r.get('regs', '?'):>4} regs stack {r.get('stack', 0):>4} spill {r.get('st', 0)}/{r.get('ld', 0)}  {n}")


if __name__ == "__main__":
    main()
