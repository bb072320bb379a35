"""Emit search specs for bitsliced field ops (see search.c)."""
import itertools
import sys

def f3_us_pats():  # unit/sign: value -> (u, s) bits; pattern int = u | s<<1
    return {0: 0b00, 1: 0b01, 2: 0b11}

def f3_ab_pats():  # value = a - b: 0=00, 1=a=1 (01 as int a|b<<1 = 1), -1 = b=1 (2)
    return {0: 0b00, 1: 0b01, 2: 0b10}

def spec(name):
    pts = []
    if name in ("f3_us_cpn", "f3_ab_cpn", "f3_ab_cpp"):
        P = f3_us_pats() if name.startswith("f3_us") else f3_ab_pats()
        for c, p, n in itertools.product(range(3), repeat=3):
            if name == "f3_ab_cpp":
                v = (c + p + n) % 3
            else:
                v = (c + p - n) % 3
            ib = P[c] | (P[p] << 2) | (P[n] << 4)
            pts.append((ib, P[v]))
        return 6, 2, pts
    if name in ("f3_us_add", "f3_us_sub", "f3_ab_add"):
        P = f3_us_pats() if "us" in name else f3_ab_pats()
        for c, p in itertools.product(range(3), repeat=2):
            v = (c + p) % 3 if "add" in name else (c - p) % 3
            pts.append((P[c] | (P[p] << 2), P[v]))
        return 4, 2, pts
    if name == "f7_add_canon_in":  # 3-bit + 3-bit -> 3-bit (mod 7, any rep: use canonical-free? unique: value mod 7 with 7 allowed?)
        raise SystemExit("not unique")
    raise SystemExit("unknown spec " + name)

ni, no, pts = spec(sys.argv[1])
print(ni, no, len(pts))
for ib, ob in pts:
    print(ib, ob)
