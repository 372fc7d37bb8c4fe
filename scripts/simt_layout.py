"""Search the shared-memory strides of the SIMT fused kernel (fused_elem_simt)
for conflict-free 64-bit accesses, and emit csrc/simt_layout.h.

Model: a warp's 64-bit shared access is served per half-warp; a half-warp
needs as many wavefronts as the largest number of DISTINCT addresses that fall
in the same 8-byte bank pair (addr mod 16, in doubles).  Cost of a layout =
total wavefronts over every shared load/store of one brick.
usage: python scripts/simt_layout.py [--check P1 Q BX BY]"""
import itertools
import sys


def wavefronts(addrs):
    w = 0
    for h in (addrs[:16], addrs[16:]):
        banks = {}
        for a in h:
            if a is None:
                continue
            banks.setdefault(a % 16, set()).add(a)
        w += max((len(s) for s in banks.values()), default=0)
    return w


def stage_cost(nitems, NT, addr_fns):
    """addr_fns: list of functions item -> address (one per access of the item)."""
    cost = 0
    for base in range(0, nitems, NT):
        for w0 in range(base, min(base + NT, nitems), 32):
            lanes = [it if it < nitems and it < base + NT else None for it in range(w0, w0 + 32)]
            for f in addr_fns:
                cost += wavefronts([None if it is None else f(it) for it in lanes])
    return cost


def layout_cost(P, Q, NE, NT, S1, SP, EB, SA, NA=2, NB=3, LXS=None):
    p = P - 1
    BX = 2 if NE >= 2 else 1
    LZ = P
    LY = p * (NE // BX) + 1
    if LXS is None:
        LXS = LY * LZ + (1 - (LY * LZ) % 2)
    T1SZ = NA * Q * S1
    cost = 0
    # S1: reads lattice (a loop), writes T1 (m, qx)
    def s1(it):
        el, r = divmod(it, P * P)
        return el, r // P, r % P
    f = []
    for a in range(P):
        f.append(lambda it, a=a: (lambda el, b, c: c + LZ * (p * (el // BX) + b) + LXS * (p * (el % BX) + a))(*s1(it)))
    for m in range(NA):
        for qx in range(Q):
            f.append(lambda it, m=m, qx=qx: (lambda el, b, c: el * EB + m * Q * S1 + qx * S1 + b * P + c)(*s1(it)))
    cost += stage_cost(NE * P * P, NT, f)
    # S2 / S2T: item (qx, c), c fastest
    def s2(it):
        el, r = divmod(it, Q * P)
        return el, r // P, r % P
    f = []
    for m in range(NA):
        for b in range(P):
            f.append(lambda it, m=m, b=b: (lambda el, qx, c: el * EB + m * Q * S1 + qx * S1 + b * P + c)(*s2(it)))
    for m in range(NB):
        for qy in range(Q):
            f.append(lambda it, m=m, qy=qy: (lambda el, qx, c: el * EB + T1SZ + m * Q * Q * SP + (qy * Q + qx) * SP + c)(*s2(it)))
    cost += 2 * stage_cost(NE * Q * P, NT, f)
    # S3: item pt; reads + writes T2 (m, c)
    f = []
    for m in range(NB):
        for c in range(P):
            f.append(lambda it, m=m, c=c: (lambda el, pt: el * EB + T1SZ + m * Q * Q * SP + pt * SP + c)(*divmod(it, Q * Q)))
    cost += 2 * stage_cost(NE * Q * Q, NT, f)
    # S1T: reads T1 (m, qx) [counted in S1 symmetric], writes ye (a)
    f = []
    for m in range(NA):
        for qx in range(Q):
            f.append(lambda it, m=m, qx=qx: (lambda el, b, c: el * EB + m * Q * S1 + qx * S1 + b * P + c)(*s1(it)))
    for a in range(P):
        f.append(lambda it, a=a: (lambda el, b, c: el * EB + T1SZ + c + P * b + SA * a)(*s1(it)))
    cost += stage_cost(NE * P * P, NT, f)
    return cost


def ideal(P, Q, NE, NT, NA=2, NB=3):
    return layout_cost(P, Q, NE, NT, 10**6, 10**5, 10**8, 10**4, NA, NB, LXS=10**7)


def search(P, Q, NE, NT, NA=2, NB=3):
    best = None
    for S1 in range(P * P, P * P + 16):
        for SP in range(P, P + 16):
            for SA in (P * P, P * P + 1):
                T1SZ = NA * Q * S1
                base = T1SZ + max(NB * Q * Q * SP, SA * P)
                for eo in range(16):
                    EB = base + eo
                    c = layout_cost(P, Q, NE, NT, S1, SP, EB, SA, NA, NB)
                    key = (c, EB)
                    if best is None or key < best[0]:
                        best = (key, (S1, SP, EB, SA))
    return best


if __name__ == "__main__":
    P, Q, NE, NT = 6, 7, 4, 224
    if len(sys.argv) > 1:
        P, Q, NE, NT = map(int, sys.argv[1:5])
    print("ideal-ish", ideal(P, Q, NE, NT))
    print(search(P, Q, NE, NT))
