"""Dynamic instruction / stall breakdown of one kernel from an ncu SASS
source export (ncu -i rep --page source --csv --print-source sass), split
into regions at every BAR.SYNC (the fused kernel's pass boundaries).
usage: sass_regions.py export.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iex = h.index("Instructions Executed")
    ist = h.index("Warp Stall Sampling (All Samples)")
    regions = [[]]
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        regions[-1].append(r)
        if "BAR.SYNC" in r[isrc] or "BAR.RED" in r[isrc]:
            regions.append([])
    tot_ex = sum(float(r[iex] or 0) for reg in regions for r in reg)
    tot_st = sum(float(r[ist] or 0) for reg in regions for r in reg)
    allops = collections.Counter()
    for k, reg in enumerate(regions):
        ex = sum(float(r[iex] or 0) for r in reg)
        stl = sum(float(r[ist] or 0) for r in reg)
        if ex / tot_ex < 0.005 and stl / tot_st < 0.005:
            continue
        ops = collections.Counter()
        for r in reg:
            s = r[isrc].strip()
            if s.startswith("@"):
                s = s.split(None, 1)[1]
            op = s.split()[0].split(".")[0]
            ops[op] += float(r[iex] or 0)
            allops[op] += float(r[iex] or 0)
        top = ", ".join(f"{o} {100 * c / ex:.0f}%" for o, c in ops.most_common(8))
        print(f"region {k:2d} [{reg[0][ia][-5:]}..{reg[-1][ia][-5:]}] {len(reg):5d} sass  "
              f"exec {100 * ex / tot_ex:5.1f}%  stalls {100 * stl / tot_st:5.1f}%  | {top}")
    print("total executed warp-instructions", int(tot_ex))
    print("all:", ", ".join(f"{o} {100 * c / tot_ex:.1f}%" for o, c in allops.most_common(20)))


if __name__ == "__main__":
    main(sys.argv[1])
