"""Event simulation of the host pipeline (csrc/host_pipeline.cu) to choose
its tiling: one H2D stream, one compute stream, one D2H stream, with PCIe
rates measured by scripts/pcie_2d_probe.py.

Two schedule families:
  grid   -- R x Nc tiles of C, operands copied in the greedy order (round-1 plan)
  grow   -- operands arrive as strips (A row blocks, B column chunks); when a
            strip lands, ONE GEMM covers that strip against everything of the
            other operand already resident (the loaded rectangle grows), and
            its C block is copied back at once.
"""
import json
import math
import sys

M = N = 32768
K = 8192
TF = 430e12          # device GEMM rate (3xFP16 pair kernel, full waves)
SLOTS = 74           # pair tiles resident at once (148 SMs / 2)

# GB/s for a 2D copy vs row bytes, with the other direction busy (filled in
# from the probe; contiguous copies use the 'contig' entry)
H2D = {"contig": 50.0}
D2H = {"contig": 52.0}


def rate(tab, row_bytes, contig=False):
    if contig or not [k for k in tab if k != "contig"]:
        return tab["contig"]
    keys = sorted(k for k in tab if k != "contig")
    if row_bytes <= keys[0]:
        return tab[keys[0]]
    if row_bytes >= keys[-1]:
        return tab[keys[-1]]
    for a, b in zip(keys, keys[1:]):
        if a <= row_bytes <= b:
            f = (math.log(row_bytes) - math.log(a)) / (math.log(b) - math.log(a))
            return tab[a] + f * (tab[b] - tab[a])


def gemm_ms(r, c):
    tiles = math.ceil(r / 256) * math.ceil(c / 256)
    waves = math.ceil(tiles / SLOTS)
    eff = tiles / (waves * SLOTS)
    return 2.0 * r * c * K / (TF * eff) * 1e3 + 0.01


def prep_ms(nbytes):
    return nbytes * 3 / 6e12 * 1e3 + 0.005   # read fp32, write 2 fp16 planes


def simulate(items, tiles_for):
    """items: [(kind 'a'|'b', start, size)] in H2D order; tiles_for(i, loaded)
    returns the C blocks [(r0, r1, c0, c1)] that item i enables."""
    t_h2d = 0.0
    t_comp = 0.0
    t_d2h = 0.0
    first_d2h = None
    for i, (kind, s0, sz) in enumerate(items):
        if kind == "a":
            nbytes = sz * K * 4
            t_h2d += nbytes / (rate(H2D, K * 4, contig=True) * 1e9) * 1e3
        else:
            nbytes = sz * K * 4
            t_h2d += nbytes / (rate(H2D, sz * 4) * 1e9) * 1e3
        t_comp = max(t_comp, t_h2d) + prep_ms(nbytes)
        for (r0, r1, c0, c1) in tiles_for(i):
            t_comp += gemm_ms(r1 - r0, c1 - c0)
            nb = (r1 - r0) * (c1 - c0) * 4
            contig = (c0 == 0 and c1 == N)
            start = max(t_d2h, t_comp)
            if first_d2h is None:
                first_d2h = start
            t_d2h = start + nb / (rate(D2H, (c1 - c0) * 4, contig) * 1e9) * 1e3
    return t_d2h, first_d2h


def grid_plan(R, Nc):
    nrb, ncb = math.ceil(M / R), math.ceil(N / Nc)
    order, na, nb = [], 0, 0
    a_bytes, b_bytes = R * K, K * Nc
    while na < nrb or nb < ncb:
        if nb == 0:
            tb = True
        elif na == 0:
            tb = False
        elif na == nrb:
            tb = True
        elif nb == ncb:
            tb = False
        else:
            tb = na / b_bytes > nb / a_bytes
        if tb:
            order.append(("b", nb * Nc, min(Nc, N - nb * Nc))); nb += 1
        else:
            order.append(("a", na * R, min(R, M - na * R))); na += 1
    return order


def grow_tiles(items):
    """the growing-rectangle schedule: strip x resident extent of the other operand"""
    out, ra, cb = [], [], []
    for kind, s0, sz in items:
        if kind == "a":
            ra.append((s0, s0 + sz))
            out.append([(s0, s0 + sz, c0, c1) for (c0, c1) in merge(cb)])
        else:
            cb.append((s0, s0 + sz))
            out.append([(r0, r1, s0, s0 + sz) for (r0, r1) in merge(ra)])
    return out


def merge(iv):
    iv = sorted(iv)
    res = []
    for a, b in iv:
        if res and res[-1][1] == a:
            res[-1] = (res[-1][0], b)
        else:
            res.append((a, b))
    return res


def grid_tiles(items, R, Nc):
    out, ra, cb = [], [], []
    for kind, s0, sz in items:
        if kind == "a":
            ra.append((s0, s0 + sz)); out.append([(s0, s0 + sz, c0, c1) for (c0, c1) in cb])
        else:
            cb.append((s0, s0 + sz)); out.append([(r0, r1, s0, s0 + sz) for (r0, r1) in ra])
    return out


def strips(total, sizes):
    out, s = [], 0
    i = 0
    while s < total:
        w = min(sizes[min(i, len(sizes) - 1)], total - s)
        out.append((s, w)); s += w; i += 1
    return out


def grow_order(a_sizes, b_sizes):
    """interleave A and B strips keeping the loaded rectangle square-ish in bytes"""
    A = [("a", s, w) for s, w in strips(M, a_sizes)]
    B = [("b", s, w) for s, w in strips(N, b_sizes)]
    order, ia, ib, la, lb = [], 0, 0, 0, 0
    while ia < len(A) or ib < len(B):
        if ib < len(B) and (ia == len(A) or lb <= la):
            order.append(B[ib]); lb += B[ib][2]; ib += 1
        else:
            order.append(A[ia]); la += A[ia][2]; ia += 1
    return order


def main():
    if len(sys.argv) > 1:
        for line in open(sys.argv[1]):
            d = json.loads(line)
            if d["other_busy"]:
                (H2D if d["dir"] == "h2d" else D2H)[d["row_bytes"]] = d["GB/s"]
        H2D["contig"] = max(v for k, v in H2D.items())
        D2H["contig"] = max(v for k, v in D2H.items())
    res = []
    for R, Nc in ((2048, 16384), (2048, 8192), (4096, 16384)):
        it = grid_plan(R, Nc)
        tl = grid_tiles(it, R, Nc)
        t, f = simulate(it, lambda i: tl[i])
        res.append(("grid", R, Nc, t, f))
    for a0 in (1024, 2048):
        for bseq in ([2048, 2048, 4096, 8192, 16384], [4096, 4096, 8192, 16384], [1024, 1024, 2048, 4096, 8192, 16384],
                     [2048], [4096], [8192], [2048, 2048, 4096, 4096, 8192]):
            for aseq in ([a0], [a0, a0, 2 * a0, 4 * a0]):
                it = grow_order(aseq, bseq)
                tl = grow_tiles(it)
                t, f = simulate(it, lambda i: tl[i])
                res.append(("grow", aseq, bseq, t, f))
    res.sort(key=lambda r: r[3])
    for r in res:
        print(f"{r[0]:5s} {str(r[1]):24s} {str(r[2]):34s} total {r[3]:6.1f} ms  first D2H {r[4]:5.1f} ms  "
              f"{2 * M * N * K / r[3] / 1e9:6.1f} TF")


if __name__ == "__main__":
    main()
