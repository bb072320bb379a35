"""Exhaustive checks of the LOP3 formulas used by the kernel (bit-level simulation)."""
import itertools

M = 1

def lop3(a, b, c, imm):
    r = 0
    for i in range(8):
        if (imm >> i) & 1:
            r |= (a if i & 4 else 1 - a) & (b if i & 2 else 1 - b) & (c if i & 1 else 1 - c)
    return r

XOR3, MAJ, AND2 = 0x96, 0xE8, 0xC0

def f3_add(xu, xs, yu, ys):
    w = lop3(xu, xs, ys, 0x61)
    return lop3(xu, yu, w, 0x7c), lop3(xs, yu, w, 0x24)

def f3_sub(xu, xs, yu, ys):
    w = lop3(xu, xs, ys, 0x61)
    return lop3(xu, yu, w, 0xbc), lop3(xs, yu, w, 0x28)

ENC = {0: (0, 0), 1: (1, 0), 2: (1, 1)}
DEC = {v: k for k, v in ENC.items()}
for x, y in itertools.product(range(3), repeat=2):
    assert DEC[f3_add(*ENC[x], *ENC[y])] == (x + y) % 3
    assert DEC[f3_sub(*ENC[x], *ENC[y])] == (x - y) % 3
print("f3 add/sub 3-LOP3 ok")

def bits(v, n): return [(v >> i) & 1 for i in range(n)]
def val(bs): return sum(b << i for i, b in enumerate(bs))

def f7_add(a, b):
    c0 = lop3(a[0], b[0], 0, AND2)
    c1 = lop3(a[1], b[1], c0, MAJ)
    co = lop3(a[2], b[2], c1, MAJ)
    C1 = lop3(a[0], b[0], co, MAJ)
    C2 = lop3(a[1], b[1], C1, MAJ)
    return [lop3(a[0], b[0], co, XOR3), lop3(a[1], b[1], C1, XOR3), lop3(a[2], b[2], C2, XOR3)]

for x, y in itertools.product(range(8), repeat=2):
    r = val(f7_add(bits(x, 3), bits(y, 3)))
    assert r % 7 == (x + y) % 7, (x, y, r)
print("f7 add 8-LOP3 ok")

def add15(a, b):
    c0 = lop3(a[0], b[0], 0, AND2)
    c1 = lop3(a[1], b[1], c0, MAJ)
    c2 = lop3(a[2], b[2], c1, MAJ)
    co = lop3(a[3], b[3], c2, MAJ)
    C1 = lop3(a[0], b[0], co, MAJ)
    C2 = lop3(a[1], b[1], C1, MAJ)
    C3 = lop3(a[2], b[2], C2, MAJ)
    return [lop3(a[0], b[0], co, XOR3), lop3(a[1], b[1], C1, XOR3), lop3(a[2], b[2], C2, XOR3), lop3(a[3], b[3], C3, XOR3)]

for x, y in itertools.product(range(16), repeat=2):
    r = val(add15(bits(x, 4), bits(y, 4)))
    assert r % 15 == (x + y) % 15, (x, y, r)
# doubling = rotate left in 4 bits (mod 15)
for x in range(16):
    b = bits(x, 4)
    assert val([b[3], b[0], b[1], b[2]]) % 15 == (2 * x) % 15
print("mod-15 add 11-LOP3 + rotate-double ok")
