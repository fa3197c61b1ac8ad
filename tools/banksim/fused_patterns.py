"""Bank-conflict counts of every shared-memory access pattern of heat_fused_axis0_kernel
(N = 1024, V = 16, P = 4) under candidate OutPair layouts."""
import sys
from banks import N, V, T, H2, hpidx, run

P = 4


def chunk(r, c):
    return c ^ ((r >> 1) & 3)


def outpair_idx(off):
    def idx(e):
        k = (e + 1) >> 1
        return (e & 1) * (H2 + off) + (k ^ ((k >> 3) & 7))
    return idx


def patterns(idx):
    res = {}
    # forward pre-read from the tile mirror (two reads per p)
    res["pre_tile"] = run(lambda t: [((m - 1) * P + chunk(m - 1, 0)) if m > 0 else None
                                     for m in (t + T * p for p in range(V))] +
                               [((N - m - 1) * P + chunk(N - m - 1, 0)) if m > 0 else None
                                for m in (t + T * p for p in range(V))])
    # post puts in the fused last stage (NSL = 256, RL = 4, BL = 4)
    NSL, RL, BL = 256, 4, 4

    def jj(t):
        out = []
        for i in range(BL // 2):
            out.append(T * i if t == 0 else t + T * i)
        for i in range(BL // 2):
            out.append(T * (BL // 2 + i) if t == 0 else NSL - (t + T * i))
        return out

    def puts(t, odd):
        a = []
        for b in range(BL):
            for q in range(RL // 2):
                k = jj(t)[b] + NSL * q
                if odd:
                    a.append(idx(2 * k - 1) if k > 0 else None)
                else:
                    a.append(idx(2 * k))
        return a
    res["post_put_odd"] = run(lambda t: puts(t, True))
    res["post_put_even"] = run(lambda t: puts(t, False))
    H = V // 2
    res["scan_get"] = run(lambda t: [idx(2 * (t * H + i)) for i in range(H)])
    # recurrence slots
    res["rec"] = run(lambda t: [t + T * i for i in range(V)])
    # inverse pre-read
    res["pre_inv"] = run(lambda t: [idx(m - 1) if m > 0 else None for m in (t + T * p for p in range(V))] +
                              [idx(N - m - 1) if m > 0 else None for m in (t + T * p for p in range(V))])
    return res


def store_copy(idx, RG):
    n = N - 1
    tot = ideal = 0
    from banks import wavefronts
    for w0 in range(0, P * n, 32):
        addrs = []
        for e in range(w0, w0 + 32):
            if e < P * n:
                q, kk = e % P, e // P
                addrs.append(q * RG + idx(kk))
            else:
                addrs.append(None)
        tot += wavefronts(addrs)
        ideal += -(-sum(a is not None for a in addrs) // 8)
    return tot, ideal


for off in (0, 4):
    idx = outpair_idx(off)
    print("odd-half offset", off)
    for k, (w, i) in patterns(idx).items():
        print(f"  {k:14s} wavefronts {w:6d} ideal {i:6d}  x{w / i:.2f}")
    for RG in (1090, 1094, 1092):
        w, i = store_copy(idx, RG)
        print(f"  store RG={RG}   wavefronts {w:6d} ideal {i:6d}  x{w / i:.2f}")

print("recurrence relayout: read OutPair(off) at e = t + T i - 1, write linear at t + T i")
for off in (0, 4):
    idx = outpair_idx(off)
    print(" off", off, "read", run(lambda t: [idx(t + T * i - 1) if t + T * i - 1 >= 0 else None
                                             for i in range(V)]),
          "write", run(lambda t: [t + T * i for i in range(V)]),
          "pre_inv linear", run(lambda t: [m if m > 0 else None for m in (t + T * p for p in range(V))] +
                                [N - m if m > 0 else None for m in (t + T * p for p in range(V))]))
