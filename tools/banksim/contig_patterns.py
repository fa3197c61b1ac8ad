"""Bank conflicts of the contiguous kernel's OutSplit staging (8-byte accesses, N = 1024,
V = 16, T = 64) under candidate layouts: current opad (e + e/16) vs even/odd split halves
with an XOR swizzle.  Run: python contig_patterns.py"""
from banks import wavefronts

N, V, T = 1024, 16, 64
H = V // 2
NSL, RL, BL = 256, 4, 4


def run8(access, nthreads=T):
    per_t = [access(t) for t in range(nthreads)]
    tot = ideal = 0
    for w in range(0, nthreads, 32):
        for i in range(len(per_t[0])):
            addrs = [per_t[t][i] for t in range(w, w + 32)]
            tot += wavefronts(addrs, size=8)
            ideal += -(-sum(a is not None for a in addrs) // 16)
    return tot, ideal


def jj(t):
    out = [T * i if t == 0 else t + T * i for i in range(BL // 2)]
    out += [T * (BL // 2 + i) if t == 0 else NSL - (t + T * i) for i in range(BL // 2)]
    return out


def layouts():
    yield "opad e+e/16", lambda e: e + e // 16
    for off in (0, 8, 16, 24):
        for sh in (3, 4):
            def f(e, off=off, sh=sh):
                k = (e + 1) >> 1
                s = k ^ ((k >> sh) & 15)
                return (e & 1) * (N // 2 + off) + s
            yield f"split off={off} swz k^((k>>{sh})&15)", f


for name, pos in layouts():
    r = {}
    r["post_put_odd"] = run8(lambda t: [pos(2 * (jj(t)[b] + NSL * q) - 1) if jj(t)[b] + NSL * q > 0 else None
                                        for b in range(BL) for q in range(RL // 2)])
    r["post_put_even"] = run8(lambda t: [pos(2 * (jj(t)[b] + NSL * q)) for b in range(BL) for q in range(RL // 2)])
    r["scan_get"] = run8(lambda t: [pos(2 * (t * H + i)) for i in range(H)])
    r["store_copy"] = run8(lambda t: [pos(e) if e < N - 1 else None for e in range(t, N, T)])
    tot = sum(v[0] for v in r.values()); ide = sum(v[1] for v in r.values())
    print(f"{name:34s} total x{tot / ide:.3f}  " + "  ".join(f"{k} x{v[0] / v[1]:.2f}" for k, v in r.items()))
