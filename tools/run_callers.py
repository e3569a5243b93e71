"""Run bench.callers() alone (cfg4 Stokes cavities, cfg5 Taylor-Green steps)
and print its JSON."""
import json, sys
sys.path.insert(0, '.')
import bench
out = bench.callers()
print(json.dumps(out))
