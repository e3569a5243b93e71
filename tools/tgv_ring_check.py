"""Run bench.box_tgv_sharded through in-process ranks (dist_box.ThreadComm)
on one GPU: exercises the bench's cfg5-on-N-GPUs code path (the timing is
not meaningful: the ranks share one device).  usage: tgv_ring_check.py world n"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1910_03032_b200 import dist_box as D  # noqa: E402

world, n = int(sys.argv[1]), int(sys.argv[2])
out = D.run_threads(world, lambda comm: bench.box_tgv_sharded(comm, n=n, steps=2))
print(json.dumps(out[0]))
