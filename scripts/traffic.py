"""Per-kernel-class DRAM traffic and time from an ncu launch list of one bench step
(`ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`):

    python scripts/traffic.py gpurun_out/launches_dram.csv > profiles/r01_traffic.json

Classes follow bench.py's kernel classes (parl_ctx_profile): gemm, head, attn_fwd,
attn_bwd, norm, loss, pack, seed (the head GEMMs fold into gemm here).  ncu replays each kernel with cold caches, so times are
serialised / cold; the DRAM bytes are the measured traffic per launch."""
import collections
import csv
import json
import sys

UNIT = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}


def klass(name, grid):
    n = name
    if "k_attn_fwd" in n:
        return "attn_fwd"
    if "k_attn_bwd" in n or "k_attn_d" in n or "k_attn_prep" in n:
        return "attn_bwd"
    if "k_gemm" in n or "splitk" in n:
        return "gemm"
    if "softmax_bwd" in n:
        return "seed"
    if "lse_combine" in n:
        return "head"
    if "grpo" in n or "advantages" in n:
        return "loss"
    if "k_pack" in n:
        return "pack"
    return "norm"


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    per = collections.defaultdict(dict)  # launch id -> metrics
    for d in data:
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        per[d["ID"]][d["Metric Name"]] = v
        per[d["ID"]]["name"] = d["Kernel Name"]
        per[d["ID"]]["grid"] = d.get("Grid Size", "")
    agg = collections.defaultdict(lambda: {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
    kern = collections.defaultdict(lambda: {"launches": 0, "time_s": 0.0, "dram_bytes": 0.0})
    for m in per.values():
        c = klass(m["name"], m["grid"])
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        for a, key in ((agg, c), (kern, m["name"].split("(")[0].replace("void ", ""))):
            a[key]["launches"] += 1
            a[key]["time_s"] += m.get("gpu__time_duration.sum", 0.0)
            a[key]["dram_bytes"] += b
    out = {"source": path, "note": "ncu cold-cache serialised replay of one C2 bench step; dram bytes = read + write",
           "classes": {k: dict(v, dram_bytes_per_launch=v["dram_bytes"] / v["launches"]) for k, v in agg.items()},
           "kernels": {k: dict(v, dram_bytes_per_launch=v["dram_bytes"] / v["launches"])
                       for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["time_s"])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
