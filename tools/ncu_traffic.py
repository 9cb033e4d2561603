"""Fold gpurun_out/traffic/<cfg>_<precision>.csv (tools/ncu_traffic.sh) into
profiles/ncu_traffic.json: per config/precision/scatter mode, the mean DRAM
read+write bytes and duration per launch of the main force kernel and of the
filter (ncu, one GPU, --clock-control none; cold-cache serialised launches)."""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ncu pipe metrics (.avg.pct_of_peak_sustained_elapsed) -> short names
PIPES = {
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64_cycles",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_elapsed": "fp64_inst",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed": "fma_cycles",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_elapsed": "fma_inst",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed": "xu_inst",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_elapsed": "alu_inst",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed": "lsu_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput",
}


def fold(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return None
    h = rows[0]
    per = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"]
        kind = "filter" if "k_filter" in name else "force"
        if kind == "force":
            # <R, Acc, G, SPEC, DET, OVF, FOREIGN>: only the main launch
            # (OVF = FOREIGN = 0), never a tier launch
            # packed: <R, Acc, SPEC, DET, OVF, FOREIGN>
            packed = "k_force_packed<" in name
            tag = "k_force_packed<" if packed else "k_force<"
            lt = name.find(tag) + len(tag)
            args = [x.strip() for x in name[lt:name.find(">", lt)].split(",")]
            o = 4 if packed else 5
            if len(args) >= o + 2 and (args[o] not in ("0", "(bool)0", "false")
                                       or args[o + 1] not in ("0", "(bool)0", "false")):
                continue
        e = per.setdefault(d["ID"], {"kind": kind, "name": name})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"%": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
                 "ms": 1e6, "usecond": 1e3, "nsecond": 1, "msecond": 1e6}.get(unit, 1)
        e[d["Metric Name"]] = v * scale
    out = {}
    for kind in ("force", "filter"):
        ks = [e for e in per.values() if e["kind"] == kind]
        if not ks:
            continue
        rd = sum(e.get("dram__bytes_read.sum", 0) for e in ks) / len(ks)
        wr = sum(e.get("dram__bytes_write.sum", 0) for e in ks) / len(ks)
        ns = sum(e.get("gpu__time_duration.sum", 0) for e in ks) / len(ks)
        out[kind] = {"kernel": ks[0]["name"][:120], "launches": len(ks), "dram_read_bytes": rd,
                     "dram_write_bytes": wr, "traffic_bytes": rd + wr, "duration_ns": ns,
                     "dram_gbps": (rd + wr) / ns if ns else None}
        pipes = {}
        for key, short in PIPES.items():
            vals = [e[key] for e in ks if key in e]
            if vals:
                pipes[short] = round(sum(vals) / len(vals) / 100.0, 4)
        if pipes:
            out[kind]["pipes_frac_of_peak"] = pipes
    return out


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "traffic")
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tab = json.load(open(dst)) if os.path.exists(dst) else {}
    for path in sorted(glob.glob(os.path.join(src, "*.csv"))):
        cfg, prec = os.path.basename(path)[:-4].rsplit("_", 1)
        res = fold(path)
        if res:
            tab[f"{cfg}/{prec}/atomic"] = res
    json.dump(tab, open(dst, "w"), indent=1, sort_keys=True)
    print(json.dumps({k: {kk: vv.get("traffic_bytes") for kk, vv in v.items()}
                      for k, v in tab.items()}, indent=1))


if __name__ == "__main__":
    main()
