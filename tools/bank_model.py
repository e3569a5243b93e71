"""Per-pass shared-memory wavefront model of sf3_fast_kernel (8-byte accesses).

For each pass we enumerate the warp-level access instructions the kernel
issues (thread -> address for every unrolled load/store) and count
wavefronts: per half-warp, max over 4-byte banks of distinct 8-byte words.
"""
import sys


def wf(addrs):
    tot = 0
    for h in (addrs[:16], addrs[16:]):
        h = [a for a in h if a is not None]
        if not h:
            continue
        cnt = {}
        for a in set(h):
            cnt[a % 16] = cnt.get(a % 16, 0) + 1
        tot += max(cnt.values())
    return tot


def ideal(addrs):
    return sum(1 for h in (addrs[:16], addrs[16:]) if any(a is not None for a in h))


def run(N, Q, NE, NT, QP=None, YP=None, ES=None, verbose=True):
    QP = QP or (Q | 1)
    YP = YP or Q * QP
    BUF = Q * YP
    ES = ES or 4 * BUF
    IX = lambda z, y, x: z * YP + y * QP + x
    passes = {}

    def pas(name, nlines, decomp, npts, addr_fn):
        w = i = 0
        for w0 in range(0, NT, 32):
            for s in range(npts):
                a = []
                for t in range(w0, w0 + 32):
                    if t < NE * nlines:
                        el, r = divmod(t, nlines)
                        a.append(el * ES + addr_fn(decomp(r), s))
                    else:
                        a.append(None)
                w += wf(a)
                i += ideal(a)
        passes[name] = passes.get(name, (0, 0))
        passes[name] = (passes[name][0] + w, passes[name][1] + i)

    # P1 x-lines (k,j): read N (gather buffer, pitch N|1), write Q
    NX = N | 1
    pas("P1 rd", N * N, lambda r: divmod(r, N), N, lambda kj, s: (kj[0] * N + kj[1]) * NX + s)
    pas("P1 wr", N * N, lambda r: divmod(r, N), Q, lambda kj, s: BUF + IX(kj[0], kj[1], s))
    # P2 y-lines (k,a)
    pas("P2 rd", N * Q, lambda r: divmod(r, Q), N, lambda ka, s: BUF + IX(ka[0], s, ka[1]))
    pas("P2 wr", N * Q, lambda r: divmod(r, Q), Q, lambda ka, s: IX(ka[0], s, ka[1]))
    # P3 z-lines (b,a): read N, write U (Q) and Gz (Q)
    pas("P3 rd", Q * Q, lambda r: divmod(r, Q), N, lambda ba, s: IX(s, ba[0], ba[1]))
    pas("P3 wr", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ba, s: (s // Q) * 3 * BUF + IX(s % Q, ba[0], ba[1]))
    # P4 paired x (c,t) + y (c,t) lines: read 2Q, write 2Q
    pas("P4 x", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ct, s: (s // Q) * BUF + IX(ct[0], ct[1], s % Q))
    pas("P4 y", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ct, s: (s // Q) * 2 * BUF + IX(ct[0], s % Q, ct[1]))
    # P5 z-columns: per c: 4 loads + 4 stores at (c, b, a)
    pas("P5", Q * Q, lambda r: divmod(r, Q), 8 * Q, lambda ba, s: (s % 4) * BUF + IX(s // 8, ba[0], ba[1]))
    # P6 paired x,y,z: 3Q reads + 3Q writes
    pas("P6 x", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ct, s: BUF + IX(ct[0], ct[1], s % Q))
    pas("P6 y", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ct, s: 2 * BUF + IX(ct[0], s % Q, ct[1]))
    pas("P6 z", Q * Q, lambda r: divmod(r, Q), 2 * Q, lambda ct, s: 3 * BUF + IX(s % Q, ct[0], ct[1]))
    # P7 z-lines: 4Q reads, N writes
    pas("P7", Q * Q, lambda r: divmod(r, Q), 4 * Q + N, lambda ba, s: (s % 4) * BUF + IX(min(s // 4, Q - 1), ba[0], ba[1]))
    # P8 y-lines (k,a): Q reads, N writes
    pas("P8", N * Q, lambda r: divmod(r, Q), Q + N, lambda ka, s: (BUF if s >= Q else 0) + IX(ka[0], s % Q, ka[1]))
    # P9 x-lines (k,j): Q reads
    pas("P9", N * N, lambda r: divmod(r, N), Q, lambda kj, s: BUF + IX(kj[0], kj[1], s))
    tw = sum(v[0] for v in passes.values())
    ti = sum(v[1] for v in passes.values())
    if verbose:
        for k, (w, i) in passes.items():
            print(f"  {k:6s}: {w:6d} wavefronts (ideal {i:6d}, x{w / max(i, 1):.2f})")
        print(f"  total {tw} (ideal {ti}, x{tw / ti:.2f})")
    return tw, ti


if __name__ == "__main__":
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = {2: (4, 64), 3: (2, 64), 4: (4, 160), 5: (2, 128), 6: (1, 96), 7: (1, 128), 8: (1, 128)}
    NE, NT = cfg[p]
    print(f"p={p} NE={NE} NT={NT} default layout")
    run(p + 1, p + 2, NE, NT)


def search(p, NE, NT):
    N, Q = p + 1, p + 2
    best = None
    for QP in (Q, Q + 1, Q + 2):
        for dYP in range(0, 5):
            YP = Q * QP + dYP
            BUF = Q * YP
            for dES in range(0, 9):
                for nb in (4,):
                    ES = nb * BUF + dES
                    w, i = run(N, Q, NE, NT, QP, YP, ES, verbose=False)
                    cost = w + 1e-3 * ES
                    if best is None or cost < best[0]:
                        best = (cost, w, i, QP, YP, ES)
    return best
