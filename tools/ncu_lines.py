"""Per CUDA-source-line stall samples / executed instructions of an .ncu-rep
(needs -lineinfo and --import-source on).  usage: ncu_lines.py rep [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    h, kern, out = None, None, {}
    for r in rows:
        if r and r[0] == "Kernel Name":
            kern = r[1]
            out[kern] = []
            continue
        if r and r[0] in ("Line", "#"):
            h = r
            continue
        if kern and h and len(r) == len(h):
            out[kern].append(r)
    if not out or not any(out.values()):
        print("unparsed; first rows:")
        for r in rows[:12]:
            print(r[:12])
        return
    for k, v in out.items():
        try:
            si = h.index("Warp Stall Sampling (All Samples)")
            ie = h.index("Instructions Executed")
        except ValueError:
            print(h)
            return
        src = h.index("Source")
        tot = sum(float(x[si] or 0) for x in v) or 1
        toti = sum(float(x[ie] or 0) for x in v) or 1
        print("==", k[:80])
        for x in sorted(v, key=lambda x: -float(x[si] or 0))[:top]:
            print(f"  L{x[0]:>5s} stall {100*float(x[si] or 0)/tot:5.1f}%  inst {100*float(x[ie] or 0)/toti:5.1f}%  {x[src].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
