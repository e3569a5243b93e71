"""Registers / stack of the fused-kernel instantiations (default launch
shapes, Helmholtz) from an object file.  usage: regs.py [obj]"""
import re
import subprocess
import sys

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_03032_b200/_obj/fb_ops.cu.o"
out = subprocess.run(["cuobjdump", "--dump-resource-usage", obj], capture_output=True,
                     text=True).stdout
want = {(3, 4, 4, 64, 10, 1), (4, 5, 4, 128, 4, 3), (5, 6, 2, 96, 4, 3), (6, 7, 2, 128, 3, 3),
        (7, 8, 1, 64, 4, 3), (8, 9, 1, 128, 4, 0), (9, 10, 1, 128, 2, 3)}
fn = None
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
        continue
    r = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if fn and r:
        k = re.search(r"sf3_fast_kernelILi(\d+)ELi(\d+)ELi2ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", fn)
        if k and tuple(map(int, k.groups())) in want:
            print(f"p={int(k.group(1)) - 1} {k.groups()} REG {r.group(1)} STACK {r.group(2)}")
        fn = None
