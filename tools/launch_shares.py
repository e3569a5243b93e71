"""Per-kernel time shares and per-degree DRAM traffic from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).

    python tools/launch_shares.py launches.csv [shares.txt] [traffic.json]
"""
import collections
import csv
import json
import re
import statistics
import sys


def load(path):
    rows = [l for l in open(path) if l.startswith('"')]
    launches = collections.OrderedDict()
    for r in csv.DictReader(rows):
        k = launches.setdefault(r["ID"], {"name": r["Kernel Name"]})
        k[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return list(launches.values())


def main(path, out_txt=None, out_json=None):
    L = load(path)
    tot = sum(k.get("gpu__time_duration.sum", 0.0) for k in L)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k in L:
        a = agg[k["name"][:90]]
        a[0] += 1
        a[1] += k.get("gpu__time_duration.sum", 0.0)
    lines = [f"{path}: {len(L)} launches (serialised, cold-ish caches; compare shares)"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f" {100 * t / tot:5.1f}% {n:4d} launches {t / n / 1e3:10.1f} us  {name}")
    txt = "\n".join(lines)
    print(txt)
    if out_txt:
        open(out_txt, "w").write(txt + "\n")
    # per-degree traffic of the fused kernel (sf3_q1 = p 1, sf3_fast_kernel<N,...> = p N-1)
    # and of the E->L sum launch that follows it
    per = collections.defaultdict(lambda: {"k_b": [], "k_t": [], "s_b": [], "s_t": []})
    last = None
    for k in L:
        m = re.search(r"sf3_fast_kernel<\(?(?:int\)?)?\s*(\d+)", k["name"])
        p = 1 if "sf3_q1" in k["name"] else (int(m.group(1)) - 1 if m else None)
        b = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        if p is not None:
            per[p]["k_b"].append(b)
            per[p]["k_t"].append(k.get("gpu__time_duration.sum", 0.0))
            last = p
        elif "scatter_slots" in k["name"] and last is not None:
            per[last]["s_b"].append(b)
            per[last]["s_t"].append(k.get("gpu__time_duration.sum", 0.0))
            last = None
    med = lambda v: statistics.median(v) if v else 0.0  # noqa: E731
    res = {str(p): {"kernel_dram_bytes": med(v["k_b"]), "scatter_dram_bytes": med(v["s_b"]),
                    "kernel_ns": med(v["k_t"]), "scatter_ns": med(v["s_t"])}
           for p, v in sorted(per.items())}
    sweep = sum(r["kernel_dram_bytes"] + r["scatter_dram_bytes"] for r in res.values())
    if out_json:
        json.dump({"source": f"{path}; medians per launch", "per_p": res,
                   "sweep_dram_bytes": sweep}, open(out_json, "w"), indent=1)
    print("sweep DRAM bytes (fused kernel + E->L sum):", sweep)


if __name__ == "__main__":
    main(*sys.argv[1:])
