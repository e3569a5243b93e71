"""Summarise an .ncu-rep: key metrics, stall reasons, top SASS stall sites, opcode mix."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.per_cycle_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed.avg.per_cycle_active', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum']


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main(rep, top=12):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:70])
        for k in KEYS:
            if k in hdr:
                print(f"   {k:62s} {r[hdr.index(k)]:>14s} {units[hdr.index(k)]}")
        vals = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    vals.append((float(r[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in vals) or 1
        print("   stalls:", ", ".join(f"{k} {100*v/tot:.0f}%" for v, k in sorted(vals, reverse=True)[:6]))
    text = run([rep, "--page", "source", "--csv", "--print-source", "sass"])
    rows = list(csv.reader(io.StringIO(text)))
    kern, data, h = None, {}, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kern = r[1]
            data[kern] = []
            continue
        if r and r[0] == "Address":
            h = r
            continue
        if kern and h and len(r) > 3:
            data[kern].append(r)
    for k, v in data.items():
        si = h.index("Warp Stall Sampling (All Samples)")
        ie = h.index("Instructions Executed")
        tot = sum(int(x[si]) for x in v) or 1
        c = collections.Counter()
        for x in v:
            src = x[1].strip()
            if src.startswith("@"):
                src = src.split(None, 1)[1]
            c[src.split()[0].split(".")[0]] += int(x[ie])
        ti = sum(c.values()) or 1
        print("==", k[:70])
        print("   opcode mix:", ", ".join(f"{op} {100*n/ti:.0f}%" for op, n in c.most_common(10)))
        print("   top stall sites:")
        for x in sorted(v, key=lambda x: -int(x[si]))[:top]:
            print(f"     {100*int(x[si])/tot:5.1f}%  {x[1].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
