import json, sys
sys.path.insert(0, '.')
import bench
out = bench.callers()
print(json.dumps(out))
