"""Print the headline, per-degree and LOR-PCG numbers of a bench.py log."""
import json
import sys

line = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d = json.loads(line)
print("value", d["value"], d["unit"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"],
      "clocks", d["clocks"])
for p, r in d["per_p"].items():
    print(f"  p={p}: {r['gdofs']:.2f} GDoF/s  full {r['hbm_frac']:.3f}  kernel {r['kernel_hbm_frac']:.3f}")
for k in ("lor_pcg", "lor_pcg_cfg3"):
    for name, r in d.get(k, {}).items():
        if isinstance(r, dict):
            print(f"  {k} {name}: its={r.get('iterations')} solve_ms={r.get('solve_ms')} "
                  f"ms/it={r.get('ms_per_iteration')} vcycle_ms={r.get('vcycle_ms')}")
