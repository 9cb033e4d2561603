"""A/B two builds of the library on the same GPU box: alternate
`TSF_LIBRARY=<a>` / `<b>` bench runs (device-resident, all precisions as
variants) R times and print the median kernel and step times per config.
usage: python tools/ab.py <lib_a> <lib_b> [rounds] [config...]
(a "lib" may carry env settings: "path+NAME=VALUE", "+NAME=VALUE" for the default library)"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, cfg):
    # lib: a library path, or "+NAME=VALUE" (the default library with an env setting)
    # "path+NAME=VALUE+NAME2=VALUE2": a library (empty: the default) with env settings
    path, *sets = lib.split("+")
    env = dict(os.environ, TSF_LIBRARY=path) if path else dict(os.environ)
    for kv in sets:
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg,
                          "--steps", "300", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, env=env, timeout=600)
    d = json.loads(out.stdout.strip().splitlines()[-1])
    r = {"double": (d["ms_per_step"], d["roofline"]["kernel_ms"])}
    for p, v in d["variants"].items():
        r[p] = (v["ms_per_step"], v["kernel_ms"])
    if d.get("md"):
        r["md"] = (d["md"]["ms_per_step"], d["md"]["ms_per_step"])
    return r


def main():
    # ab.py <lib_a> <lib_b> [rounds] [config...], or
    # ab.py --libs a,b,c[,...] [rounds] [config...] (any number of variants)
    argv = sys.argv[1:]
    if argv[0] == "--libs":
        libs = argv[1].split(",")
        argv = argv[2:]
    else:
        libs = argv[:2]
        argv = argv[2:]
    rounds = int(argv[0]) if argv else 3
    cfgs = argv[1:] or ["si2m"]
    for cfg in cfgs:
        res = {lib: [] for lib in libs}
        for _ in range(rounds):
            for lib in libs:
                res[lib].append(run(lib, cfg))
        for prec in [p for p in ("double", "mixed", "single", "md") if p in res[libs[0]][0]]:
            line = [cfg, prec]
            for lib in libs:
                step = statistics.median(r[prec][0] for r in res[lib])
                kern = statistics.median(r[prec][1] for r in res[lib])
                line.append(f"{os.path.basename(lib) or 'default'}: step {step:.4f} kernel {kern:.4f}")
            print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
