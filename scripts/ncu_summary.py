"""Summarise ncu output for profiles/:
   python scripts/ncu_summary.py launches <launches.csv> > profiles/rNN_launches.md
   python scripts/ncu_summary.py report <prof.ncu-rep>   > profiles/rNN_<kernel>.md"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def launches(path, by_grid=False):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("parl_gpu::", "")
        name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        if by_grid:
            name += " " + d.get("Grid Size", "")
        us = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"# launch list: {path}\n\nncu `--metrics gpu__time_duration.sum --clock-control none` "
          f"(cold-cache, serialised; compare shares, not absolutes). {len(data)} launches, {tot/1e3:.2f} ms total.\n")
    print("| kernel | launches | total ms | share | mean us |\n|---|---:|---:|---:|---:|")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {us/1e3:.3f} | {100*us/tot:.1f}% | {us/n:.1f} |")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full: {path}\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## `{d.get('Kernel Name', '?')[:120]}`\n\n| metric | value | unit |\n|---|---:|---|")
        for k in WANT:
            if k in d:
                print(f"| {k} | {d[k]} | {u.get(k, '')} |")
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], by_grid="--by-grid" in sys.argv)
    else:
        report(sys.argv[2])
