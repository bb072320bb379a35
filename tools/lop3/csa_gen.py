"""Generate (and verify) the carry-save accumulation networks of the M4RM kernel.

For F7 (mod 7, 3 columns) and F5 (accumulated mod 15, 4 columns) the per-(row, k-block)
update C += x + 2y + 4z is one multi-operand addition in carry-save form: full adders (xor3 +
majority = 2 LOP3) move bits between columns, and a carry out of the top column re-enters
column 0 (2^n == 1 mod 2^n - 1).  The plan (which column each adder works on) comes from
csa_plan.py; this script picks the operand bits (earliest-ready first), emits the CUDA
function, and checks it lane-exactly on random words.  For F5, 4z is replaced by -z (4 == -1
mod 5): -z = ~z - 8 in 4-bit one's complement, so the complemented bits enter as LOP3 input
inversions and the constant -8 per block is pre-paid when the accumulator is initialised.
"""
import random

XOR3_TT = lambda a, b, c: a ^ b ^ c          # noqa: E731
MAJ_TT = lambda a, b, c: (a & b) | (a & c) | (b & c)  # noqa: E731


def lut(fn, inv):
    """LOP3 immediate of fn(a, b, c) with inputs inverted per inv = (ia, ib, ic)."""
    code = 0
    for i in range(8):
        a, b, c = (i >> 2) & 1, (i >> 1) & 1, i & 1
        a ^= inv[0]
        b ^= inv[1]
        c ^= inv[2]
        if fn(a, b, c):
            code |= 1 << i
    return code


def generate(name, ncols, state, inputs, plan, cap):
    """state/inputs: list of (col, varname, inverted).  Returns (code lines, final state)."""
    cols = [[] for _ in range(ncols)]  # entries: (depth, expr, inverted)
    for col, v, inv in state + inputs:
        cols[col].append((0, v, inv))
    lines, tmp = [], [0]

    def fresh():
        tmp[0] += 1
        return f"t{tmp[0]}"

    for kind, c in plan:
        cols[c].sort(key=lambda e: e[0])
        need = 3 if kind == "FA" else 2
        ops = [cols[c].pop(0) for _ in range(need)]
        d = max(o[0] for o in ops) + 1
        if kind == "HA":
            ops.append((0, "0u", 0))
        names = [o[1] for o in ops]
        inv = tuple(o[2] for o in ops)
        s, k = fresh(), fresh()
        lines.append(f"const u32 {s} = lop3<0x{lut(XOR3_TT, inv):02x}>({', '.join(names)});")
        lines.append(f"const u32 {k} = lop3<0x{lut(MAJ_TT, inv):02x}>({', '.join(names)});")
        cols[c].append((d, s, 0))
        cols[(c + 1) % ncols].append((d, k, 0))
    for c in range(ncols):
        assert len(cols[c]) <= cap[c], (name, c, cols[c])
    depth = max(e[0] for col in cols for e in col)
    return lines, [[e[1] for e in col] for col in cols], depth


def simulate(lines, env):
    env = dict(env)
    for ln in lines:
        lhs = ln.split("=")[0].split()[-1]
        imm = int(ln.split("<0x")[1][:2], 16)
        args = [a.strip() for a in ln.split("(")[1].split(")")[0].split(",")]
        vals = [0 if a == "0u" else env[a] for a in args]
        r = 0
        for i in range(8):
            if (imm >> i) & 1:
                a = vals[0] if i & 4 else ~vals[0]
                b = vals[1] if i & 2 else ~vals[1]
                cc = vals[2] if i & 1 else ~vals[2]
                r |= a & b & cc
        env[lhs] = r & ((1 << 64) - 1)
    return env


def lanes(env, names_by_col, lane):
    return sum(((env[n] >> lane) & 1) << col for col, names in enumerate(names_by_col) for n in names if n != "0u")


def check(name, ncols, modulus, lines, state_names, final, in_names, coef):
    M = (1 << ncols) - 1
    for _ in range(200):
        env = {v: random.getrandbits(64) for v in state_names + in_names}
        out = simulate(lines, env)
        for lane in range(64):
            before = sum(((env[v] >> lane) & 1) << c for c, v in state_cols(state_names, ncols))
            add = 0
            for (v, w) in coef:
                add += ((env[v] >> lane) & 1) * w
            after = sum(((out[n] >> lane) & 1) << c for c, names in enumerate(final) for n in names)
            assert (after - before - add) % modulus == 0, (name, lane)
    return True


def state_cols(state_names, ncols):
    return [(int(v.split("_")[1]), v) for v in state_names]


def f7():
    state = [(0, "q_0", 0), (0, "k_0", 0), (1, "q_1", 0), (2, "q_2", 0)]
    inputs = [(0, "x0", 0), (1, "x1", 0), (2, "x2", 0),      # x
              (1, "y0", 0), (2, "y1", 0), (0, "y2", 0),      # 2y mod 7
              (2, "z0", 0), (0, "z1", 0), (1, "z2", 0)]      # 4z mod 7
    plan = [("FA", 0), ("FA", 0), ("FA", 1), ("FA", 2), ("FA", 2), ("FA", 0), ("FA", 1), ("FA", 1), ("FA", 2)]
    lines, final, depth = generate("f7", 3, state, inputs, plan, (2, 1, 1))
    coef = [("x0", 1), ("x1", 2), ("x2", 4), ("y0", 2), ("y1", 4), ("y2", 8), ("z0", 4), ("z1", 8), ("z2", 16)]
    check("f7", 3, 7, lines, ["q_0", "k_0", "q_1", "q_2"], final, [v for _, v, _ in inputs], coef)
    return lines, final, depth


def f5():
    state = [(0, "q_0", 0), (1, "q_1", 0), (2, "q_2", 0), (2, "k_2", 0), (3, "q_3", 0)]
    inputs = [(0, "x0", 0), (1, "x1", 0), (2, "x2", 0),      # x
              (1, "y0", 0), (2, "y1", 0), (3, "y2", 0),      # 2y
              (0, "z0", 1), (1, "z1", 1), (2, "z2", 1)]      # ~z = -z - 8 (mod 15) == 4z - 8 (mod 5)
    plan = [("FA", 0), ("FA", 1), ("FA", 1), ("FA", 2), ("FA", 2), ("FA", 2), ("FA", 3), ("FA", 3), ("FA", 0), ("HA", 1)]
    lines, final, depth = generate("f5", 4, state, inputs, plan, (1, 1, 2, 1))
    # value identity mod 5: after == before + x + 2y + 4z - 8  (mod 5): check with coefficient
    # for the complemented bits: (1 - z_i) * 2^i summed = 7 - z  ->  -z - 8 + 15 ... verify mod 5
    M = 15
    for _ in range(200):
        names = ["q_0", "q_1", "q_2", "k_2", "q_3", "x0", "x1", "x2", "y0", "y1", "y2", "z0", "z1", "z2"]
        env = {v: random.getrandbits(64) for v in names}
        out = simulate(lines, env)
        for lane in range(64):
            b = lambda v: (env[v] >> lane) & 1  # noqa: E731
            before = b("q_0") + 2 * b("q_1") + 4 * b("q_2") + 4 * b("k_2") + 8 * b("q_3")
            x = b("x0") + 2 * b("x1") + 4 * b("x2")
            y = b("y0") + 2 * b("y1") + 4 * b("y2")
            z = b("z0") + 2 * b("z1") + 4 * b("z2")
            after = sum(((out[n] >> lane) & 1) << c for c, ns in enumerate(final) for n in ns)
            assert (after - (before + x + 2 * y + (7 - z))) % M == 0
            assert (after - (before + x + 2 * y + 4 * z - 8)) % 5 == 0
    return lines, final, depth


def emit(fname, args, lines, final, assign):
    out = [f"__device__ __forceinline__ void {fname}({args}) {{"]
    out += ["  " + ln for ln in lines]
    for dst, src in assign(final):
        out.append(f"  {dst} = {src};")
    out.append("}")
    return "\n".join(out)


if __name__ == "__main__":
    random.seed(1)
    l7, fin7, d7 = f7()
    l5, fin5, d5 = f5()
    print(f"// f7: {len(l7)} LOP3, depth {d7} full adders; final columns {fin7}")
    print(f"// f5: {len(l5)} LOP3, depth {d5} full adders; final columns {fin5}")
    print("\n".join(l7))
    print("\n".join(l5))
