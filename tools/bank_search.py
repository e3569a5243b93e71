"""Search the work-buffer pitches (x-row pitch, z-plane pitch, element pad) of
the fused kernel that minimise shared-memory wavefronts (bank_model.py's
access model); produced the SF3Pitch tables in csrc/sf3_fast.cuh."""
import itertools, sys


def wf_half(h):
    h = [a for a in h if a is not None]
    if not h:
        return 0
    banks = {}
    for a in set(h):
        k = a % 16
        banks[k] = banks.get(k, 0) + 1
    return max(banks.values())


def wavefronts(addrs):
    return wf_half(addrs[:16]) + wf_half(addrs[16:])


def lines(kind, dims, order):
    """Return list of (base_fn(point index along line)) for each line.
    kind: 'x','y','z' contraction axis; dims=(Z,Y,X) extents of the line-index axes;
    order: which of the two non-contracted axes is fastest."""
    Z, Y, X = dims
    out = []
    if kind == 'x':
        a, b = (Y, Z)  # line axes (y,z)
        it = [(z, y) for z in range(Z) for y in range(Y)] if order == 0 else \
             [(z, y) for y in range(Y) for z in range(Z)]
        return [('x', z, y) for z, y in it]
    if kind == 'y':
        it = [(z, x) for z in range(Z) for x in range(X)] if order == 0 else \
             [(z, x) for x in range(X) for z in range(Z)]
        return [('y', z, x) for z, x in it]
    it = [(y, x) for y in range(Y) for x in range(X)] if order == 0 else \
         [(y, x) for x in range(X) for y in range(Y)]
    return [('z', y, x) for y, x in it]


def addr(line, s, QP, YP):
    k, u, v = line
    if k == 'x':
        z, y = u, v
        return z * YP + y * QP + s
    if k == 'y':
        z, x = u, v
        return z * YP + s * QP + x
    y, x = u, v
    return s * YP + y * QP + x


def cost_pass(kind, dims, npts, order, QP, YP, ES, NE, NT):
    L = lines(kind, dims, order)
    nl = len(L)
    tot = 0
    for w0 in range(0, NT, 32):
        for s in range(npts):
            a = []
            for t in range(w0, w0 + 32):
                if t < NE * nl:
                    el, r = divmod(t, nl)
                    a.append(el * ES + addr(L[r], s, QP, YP))
                else:
                    a.append(None)
            tot += wavefronts(a)
    return tot


def kernel_passes(N, Q):
    # (kind, line-axis extents (Z,Y,X) of the array being accessed, points per line)
    return [
        ('x', (N, N, None), N), ('x', (N, N, None), Q),      # X pass read/write
        ('y', (N, None, Q), N), ('y', (N, None, Q), Q),      # Y pass
        ('z', (None, Q, Q), N), ('z', (None, Q, Q), Q),      # Z pass + store U
        ('x', (Q, Q, None), Q), ('x', (Q, Q, None), Q),      # DX read/write
        ('y', (Q, None, Q), Q), ('y', (Q, None, Q), Q),      # DY
        ('z', (None, Q, Q), Q), ('z', (None, Q, Q), Q), ('z', (None, Q, Q), Q),  # PW g0 g1 + V
        ('x', (Q, Q, None), Q), ('x', (Q, Q, None), Q),      # DX^T
        ('y', (Q, None, Q), Q), ('y', (Q, None, Q), Q),      # DY^T
        ('z', (None, Q, Q), Q), ('z', (None, Q, Q), Q), ('z', (None, Q, Q), Q), ('z', (None, Q, Q), N),
        ('y', (N, None, Q), Q), ('y', (N, None, Q), N),      # Y^T
        ('x', (N, N, None), Q),                              # X^T read
    ]


def total(N, Q, NE, NT, QP, YP, ES, orders):
    tot = ideal = 0
    for kind, dims, npts in kernel_passes(N, Q):
        d = tuple(1 if v is None else v for v in dims)
        tot += cost_pass(kind, d, npts, orders[kind], QP, YP, ES, NE, NT)
        nl = d[0] * d[1] * d[2]
        act = min(NE * nl, NT)
        ideal += npts * sum(min(2, (min(32, act - w0) + 15) // 16) for w0 in range(0, act, 32))
    return tot, ideal


if __name__ == "__main__":
    cfg = {1: (28, 256), 2: (16, 256), 3: (10, 256), 4: (4, 160), 5: (3, 160),
           6: (2, 128), 7: (1, 96), 8: (1, 128)}
    for p in [int(a) for a in sys.argv[1:]] or range(1, 9):
        N, Q = p + 1, p + 2
        NE, NT = cfg[p]
        best = None
        for QP in range(Q, Q + 3):
            for YP in range(Q * QP, Q * QP + 4):
                for ESx in range(0, 9):
                    ES = 3 * Q * YP + ESx
                    for ox, oy, oz in itertools.product((0, 1), repeat=3):
                        o = {'x': ox, 'y': oy, 'z': oz}
                        w, i = total(N, Q, NE, NT, QP, YP, ES, o)
                        if best is None or w < best[0]:
                            best = (w, i, QP, YP, ES, o)
        base = total(N, Q, NE, NT, Q | 1, Q * (Q | 1), 3 * Q * Q * (Q | 1), {'x': 0, 'y': 0, 'z': 0})
        print(f"p={p} NE={NE}: base {base[0]/base[1]:.2f}x  best {best[0]/best[1]:.2f}x "
              f"QP={best[2]} YP={best[3]} ES={best[4]} orders={best[5]}", flush=True)
