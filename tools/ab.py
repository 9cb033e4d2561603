"""A/B two builds of the library on the same GPU box: alternate
`TSF_LIBRARY=<a>` / `<b>` bench runs (device-resident, all precisions as
variants) R times and print the median kernel and step times per config.
usage: python tools/ab.py <lib_a> <lib_b> [rounds] [config...]
(a "lib" may also be "+NAME=VALUE": the default library with that env setting)"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, cfg):
    # lib: a library path, or "+NAME=VALUE" (the default library with an env setting)
    if lib.startswith("+"):
        k, v = lib[1:].split("=", 1)
        env = dict(os.environ, **{k: v})
    else:
        env = dict(os.environ, TSF_LIBRARY=lib) if lib else dict(os.environ)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg,
                          "--steps", "300", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, env=env, timeout=600)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    r = {"double": (d["ms_per_step"], d["roofline"]["kernel_ms"])}
    for p, v in d["variants"].items():
        r[p] = (v["ms_per_step"], v["kernel_ms"])
    return r


def main():
    a, b = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    cfgs = sys.argv[4:] or ["si2m"]
    for cfg in cfgs:
        res = {a: [], b: []}
        for _ in range(rounds):
            for lib in (a, b):
                res[lib].append(run(lib, cfg))
        for prec in ("double", "mixed", "single"):
            line = [cfg, prec]
            for lib in (a, b):
                step = statistics.median(r[prec][0] for r in res[lib])
                kern = statistics.median(r[prec][1] for r in res[lib])
                line.append(f"{os.path.basename(lib) or 'default'}: step {step:.4f} kernel {kern:.4f}")
            print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
