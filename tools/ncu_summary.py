"""Summarise an ncu --csv launch list (gpu__time_duration.sum and optional
dram__bytes_{read,write}.sum) per kernel: launches, total time, DRAM bytes."""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(lines))


def main(path):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    tscale = {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in load(path):
        k = r["Kernel Name"].split("(")[0]
        a = agg[k]
        v = float(r["Metric Value"].replace(",", ""))
        m, u = r["Metric Name"], r["Metric Unit"]
        if m == "gpu__time_duration.sum":
            a[0] += 1
            a[1] += v * tscale[u]
        elif m.startswith("dram__bytes_read"):
            a[2] += v * bscale[u]
        elif m.startswith("dram__bytes_write"):
            a[3] += v * bscale[u]
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'read GB':>8s} {'write GB':>8s} {'GB/s':>7s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        bw = (a[2] + a[3]) / (a[1] * 1e-6) / 1e9 if a[1] else 0
        print(f"{k[:34]:34s} {a[0]:8d} {a[1] / 1e3:10.1f} {100 * a[1] / tot:5.1f}% {a[2] / 1e9:8.2f} {a[3] / 1e9:8.2f} {bw:7.0f}")
    print(f"total {tot / 1e3:.1f} ms")


if __name__ == "__main__":
    main(sys.argv[1])


def traffic_json(path, n_fact, n_solve, out):
    """Per-unit DRAM traffic of the factorisation and solve kernel classes from
    a tools/profile_step.py capture (n_fact factorisations, n_solve
    pole-solves), written for bench.py's roofline.traffic."""
    import json
    agg = collections.defaultdict(float)
    bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in load(path):
        if r["Metric Name"].startswith("dram__bytes"):
            agg[r["Kernel Name"].split("(")[0]] += float(r["Metric Value"].replace(",", "")) * bscale[r["Metric Unit"]]
    fac = sum(v for k, v in agg.items() if any(s in k for s in ("gemm", "extend_add", "diag", "scatter_A", "trsm")))
    sol = sum(v for k, v in agg.items() if any(s in k for s in ("k_fwd", "k_bwd")))
    json.dump({"source": path, "factor_bytes_per_pole": fac / n_fact,
               "solve_bytes_per_pole_solve": sol / n_solve,
               "note": "dram__bytes_read.sum + dram__bytes_write.sum summed over the kernel class, "
                       "tools/profile_step.py at C4 (16 factorisations, forward + J v + J^T w = 3 "
                       "multi-RHS solves per pole)"}, open(out, "w"), indent=1)
