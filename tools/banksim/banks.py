"""Shared-memory bank-conflict model for the half-length DST kernels' access patterns.

Model (sm_100, 32 banks x 4 B): a warp's 16-byte accesses run in quarter-warp phases (lanes
8q..8q+7), 8-byte accesses in half-warp phases; a phase costs as many wavefronts as the most
loaded 16-byte (8-byte) bank group has distinct addresses.  Addresses are in units of the
access size.  Used offline to choose swizzles (K2b)."""
from collections import defaultdict

N, V = 1024, 16
T = N // V
H2 = N // 2


def hpidx(i):
    return i ^ (((i >> 3) ^ (i >> 6)) & 7)


def wavefronts(addrs, size=16):
    """addrs: list of 32 addresses (units of `size` bytes; None = inactive lane)."""
    per_phase = 8 if size == 16 else 16
    groups = 8 if size == 16 else 16
    wf = 0
    for ph in range(0, 32, per_phase):
        g = defaultdict(set)
        for a in addrs[ph:ph + per_phase]:
            if a is not None:
                g[a % groups].add(a)
        wf += max((len(s) for s in g.values()), default=0)
    return wf


def run(access, nthreads=T):
    """access(t) -> list of addresses (one per instruction); returns (wavefronts, ideal)."""
    per_t = [access(t) for t in range(nthreads)]
    ninstr = len(per_t[0])
    tot = ideal = 0
    for w in range(0, nthreads, 32):
        for i in range(ninstr):
            addrs = [per_t[t][i] for t in range(w, w + 32)]
            tot += wavefronts(addrs)
            act = sum(a is not None for a in addrs)
            ideal += -(-act // 8)
    return tot, ideal
