"""Design model of the bit-sliced FHP-III collision (development tool).

Every quantity is a "word" of independent bits (a Python int used as a
bit-vector); evaluating with 1-bit values gives the per-site rule, with
32-bit values the bit-sliced kernel. The same formulas are transcribed into
paper_1208_2428_b200/csrc/fhpg_fhp3_logic.cuh. This script checks, over all
128 fluid states and both chiralities: mass and momentum conservation,
collision saturation (every state whose (mass, momentum) class has another
member changes), rotation equivariance, mirror <-> chirality symmetry, and
that the dep formula equals "outcome depends on chirality"; it also counts
the boolean operations.

    python tools/fhp3_logic_model.py
"""
import itertools

FULL = 1  # 1-bit words when used per site

PX = [-1, 1, 2, 1, -1, -2]
PY = [1, 1, 0, -1, -1, 0]


class Ops:
    n = 0


def NOT(x):
    return ~x & FULL


def op(v):
    Ops.n += 1
    return v & FULL


def collide(a, r, c):
    """a: 6 mover words, r: rest, c: chirality. Returns (out movers, out rest, dep)."""
    # axis signals
    O = [op(a[i] ^ a[i + 3]) for i in range(3)]
    P = [op(a[i] & a[i + 3]) for i in range(3)]
    no0 = op(NOT(O[0] | O[1] | O[2]))
    no1 = op((O[0] ^ O[1] ^ O[2]) & NOT(O[0] & O[1] & O[2]))
    no2 = op((O[0] & O[1] | O[1] & O[2] | O[0] & O[2]) & NOT(O[0] & O[1] & O[2]))
    no3 = op(O[0] & O[1] & O[2])
    np0 = op(NOT(P[0] | P[1] | P[2]))
    np1 = op((P[0] ^ P[1] ^ P[2]) & NOT(P[0] & P[1] & P[2]))
    np2 = op((P[0] & P[1] | P[1] & P[2] | P[0] & P[2]) & NOT(P[0] & P[1] & P[2]))
    # momentum direction one-hot for |p| = 1 states:
    #   one odd axis: its occupied direction; two odd axes at 120 deg:
    #   the direction between them (its own axis is not odd).
    m = []
    for k in range(6):
        single = op(no1 & a[k] & NOT(a[(k + 3) % 6]))
        between = op(no2 & a[(k - 1) % 6] & NOT(a[(k + 2) % 6]))
        between = op(between & a[(k + 1) % 6] & NOT(a[(k + 4) % 6]))
        m.append(op(single | between))
    g = op(m[0] | m[1] | m[2])
    g = op(g | m[3] | m[4])
    g = op(g | m[5])  # site is in a |p|=1 class candidate
    # roles (signatures (n_odd, n_pair, rest)):
    #  type C: A=(2,0,0)  B=(1,0,1)   dual: ~A=(2,1,1)  ~B=(1,2,0)
    #  type D: X=(1,1,0)  Y=(2,0,1)   dual: ~X=(1,1,1)  ~Y=(2,1,0)
    nr = NOT(r)
    rA = op(g & no2 & np0 & nr)
    rB = op(g & no1 & np0 & r)
    rAd = op(g & no2 & np1 & r)
    rBd = op(g & no1 & np2 & nr)
    rX = op(g & no1 & np1 & nr)
    rY = op(g & no2 & np0 & r)
    rXd = op(g & no1 & np1 & r)
    rYd = op(g & no2 & np1 & nr)
    E = [op(NOT(a[i] | a[i + 3])) for i in range(3)]
    # X+: pair on the axis after the odd one; for a dual, the EMPTY axis is.
    xplus = op((O[0] & P[1]) | (O[1] & P[2]) | (O[2] & P[0]))
    xplus_d = op((O[0] & E[1]) | (O[1] & E[2]) | (O[2] & E[0]))

    def rot(v, d):
        return [v[(k - d) % 6] for k in range(6)]  # out_k = v_{k-d}

    def orr(*vs):
        out = []
        for k in range(6):
            acc = 0
            for v in vs:
                acc |= v[k]
            out.append(op(acc))
        return out

    md = rot(m, 3)  # the original-class direction of a dual site
    S0 = m
    S15 = orr(rot(m, 1), rot(m, 5))
    S052 = orr(m, rot(m, 5), rot(m, 2))
    S014 = orr(m, rot(m, 1), rot(m, 4))
    D0 = md
    D15 = orr(rot(md, 1), rot(md, 5))
    D052 = orr(md, rot(md, 5), rot(md, 2))
    D014 = orr(md, rot(md, 1), rot(md, 4))
    # chirality-0 cycle X+ -> X- -> Y -> X+, chirality 1 the reverse
    xp = xplus
    xm = NOT(xplus)
    xpd = xplus_d
    xmd = NOT(xplus_d)
    nc = NOT(c)
    # orig roles -> target set
    sel_S0 = op(rA)
    sel_S15 = op(rB | rX & (xp & c | xm & nc))
    sel_S052 = op(rX & xp & nc | rY & c)
    sel_S014 = op(rX & xm & c | rY & nc)
    sel_D0 = op(rAd)
    sel_D15 = op(rBd | rXd & (xpd & c | xmd & nc))
    sel_D052 = op(rXd & xpd & nc | rYd & c)
    sel_D014 = op(rXd & xmd & c | rYd & nc)
    coll = op(sel_S0 | sel_S15 | sel_S052 | sel_S014)
    colld = op(sel_D0 | sel_D15 | sel_D052 | sel_D014)
    out_mag1 = []
    for k in range(6):
        v = op(sel_S0 & S0[k] | sel_S15 & S15[k] | sel_S052 & S052[k] | sel_S014 & S014[k])
        vd = op(sel_D0 & D0[k] | sel_D15 & D15[k] | sel_D052 & D052[k] | sel_D014 & D014[k])
        out_mag1.append(op(v | colld & NOT(vd)))
    # rest of a |p|=1 outcome: A->B, X->Y, Y... (r = 1 for targets B, Y; dual: complement)
    r_mag1 = op(rA | rX & (xp & c | xm & nc) | rBd | rXd & NOT(xpd & c | xmd & nc) | rYd)
    # type A: zero momentum (no odd axis): rotate by +60 (c=1) / -60 (c=0)
    rotA = [op(c & a[(k - 1) % 6] | nc & a[(k + 1) % 6]) for k in range(6)]
    # type B: symmetric triples (all axes odd, alternating): complement movers
    tri = op(no3 & NOT(a[0] ^ a[2]) & NOT(a[2] ^ a[4]))
    mag1 = op(coll | colld)
    out = []
    for k in range(6):
        v = op(no0 & rotA[k] | tri & NOT(a[k]))
        v = op(v | mag1 & out_mag1[k])
        keep = op(NOT(no0 | tri | mag1))
        out.append(op(v | keep & a[k]))
    out_r = op(mag1 & r_mag1 | NOT(mag1) & r)
    dep = op(no0 & NOT(np0 | (P[0] & P[1] & P[2])) | rX | rY | rXd | rYd)
    return out, out_r, dep


def state_bits(s):
    return [(s >> k) & 1 for k in range(6)], (s >> 6) & 1


def apply(s, ch):
    a, r = state_bits(s)
    out, out_r, dep = collide(a, r, ch)
    return sum(out[k] << k for k in range(6)) | (out_r << 6), dep


def momentum(s):
    return (sum(PX[k] for k in range(6) if s >> k & 1), sum(PY[k] for k in range(6) if s >> k & 1))


def mass(s):
    return bin(s & 0x7F).count("1")


def rot_state(s, d):
    m = s & 0x3F
    d %= 6
    return (s & 0xC0) | (((m << d) | (m >> (6 - d))) & 0x3F)


MIRROR = [4, 3, 2, 1, 0, 5]  # y -> -y: NW<->SW, NE<->SE


def mirror(s):
    o = s & 0xC0
    for k in range(6):
        if s >> k & 1:
            o |= 1 << MIRROR[k]
    return o


def main():
    from collections import defaultdict
    classes = defaultdict(list)
    for s in range(128):
        classes[(mass(s),) + momentum(s)].append(s)
    size = {s: len(classes[(mass(s),) + momentum(s)]) for s in range(128)}
    table = [[0] * 128 for _ in range(2)]
    bad = 0
    for ch in (0, 1):
        for s in range(128):
            o, dep = apply(s, ch)
            table[ch][s] = o
            if mass(o) != mass(s) or momentum(o) != momentum(s):
                print(f"conservation violated s={s:07b} ch={ch} -> {o:07b}")
                bad += 1
            if size[s] > 1 and o == s:
                print(f"not saturated s={s:07b} ch={ch} class size {size[s]}")
                bad += 1
    for ch in (0, 1):
        for s in range(128):
            if table[ch][rot_state(s, 1)] != rot_state(table[ch][s], 1):
                print(f"rotation equivariance broken s={s:07b} ch={ch}")
                bad += 1
    for s in range(128):
        if table[1][mirror(s)] != mirror(table[0][s]):
            print(f"mirror/chirality broken s={s:07b}")
            bad += 1
    for ch in (0, 1):
        if sorted(table[ch]) != list(range(128)):
            print(f"chirality {ch} slice is not a permutation")
            bad += 1
    for s in range(128):
        _, dep = apply(s, 0)
        if dep != int(table[0][s] != table[1][s]):
            print(f"dep formula wrong s={s:07b}: {dep} vs {table[0][s] != table[1][s]}")
            bad += 1
    changed = sum(1 for s in range(128) if table[0][s] != s or table[1][s] != s)
    ndep = sum(1 for s in range(128) if table[0][s] != table[1][s])
    Ops.n = 0
    apply(0, 0)
    print(f"violations: {bad}; colliding states: {changed}; chirality-dependent: {ndep}; "
          f"boolean ops (unfused, per word): {Ops.n}")
    return table, bad


if __name__ == "__main__":
    main()
