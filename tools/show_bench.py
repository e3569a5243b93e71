import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d["value"], d["roofline"]["frac"], d.get("clocks"))
for p,v in d["per_p"].items(): print(p, v["gdofs"], v["hbm_frac"], v["kernel_hbm_frac"])
