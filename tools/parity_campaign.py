"""Randomized parity campaign on the GPU: random fields, shapes (up to tens of thousands of rows
and columns, ragged), k and plans (auto, or forced onto the schedule-5 / schedule-6 / fused
variants), each product compared exactly with an fp32 cuBLAS product reduced mod p (exact:
partial sums stay below 2^24; GF(4) by its closed form), plus the canonical-pattern check.
python tools/parity_campaign.py [cases] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

FIELDS = {"f3": (sg.F3, 3), "f5": (sg.F5, 5), "f7": (sg.F7, 7), "gf4": (sg.GF4, None), "f2": (sg.F2, 2),
          "gf8": (sg.GF8, None), "z4": (sg.Z4, 4), "z8": (sg.Z8, 8)}
TM_RT = {"f3": 32, "gf4": 32, "z4": 32, "f2": 32, "f5": 16, "f7": 16, "gf8": 16, "z8": 16}  # schedule-6 row-slots


def exact(fname, A, B):
    torch.backends.cuda.matmul.allow_tf32 = False
    if fname == "gf4":
        a0, a1, b0, b1 = (A & 1).float(), (A >> 1).float(), (B & 1).float(), (B >> 1).float()
        p11 = a1 @ b1
        c0 = torch.remainder(a0 @ b0 + p11, 2)
        c1 = torch.remainder(a0 @ b1 + a1 @ b0 + p11, 2)
        return (c0.to(torch.uint8) | (c1.to(torch.uint8) << 1))
    if fname == "gf8":  # F2[x] / (x^3 + x + 1): x^3 = x + 1, x^4 = x^2 + x
        a = [((A >> i) & 1).float() for i in range(3)]
        b = [((B >> i) & 1).float() for i in range(3)]
        d = [None] * 5
        for i in range(3):
            for j in range(3):
                t = a[i] @ b[j]
                d[i + j] = t if d[i + j] is None else d[i + j] + t
        c0 = torch.remainder(d[0] + d[3], 2)
        c1 = torch.remainder(d[1] + d[3] + d[4], 2)
        c2 = torch.remainder(d[2] + d[4], 2)
        return c0.to(torch.uint8) | (c1.to(torch.uint8) << 1) | (c2.to(torch.uint8) << 2)
    return torch.remainder(A.float() @ B.float(), FIELDS[fname][1]).to(torch.uint8)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    dev = torch.device("cuda", 0)
    t0, bad, ran = time.time(), 0, 0
    for it in range(cases):
        fname = list(FIELDS)[it % len(FIELDS)]
        f, p = FIELDS[fname]
        m = int(rng.choice([1, 33, 255, 1024, 2047, 4096, 5000, 8192, 8200, 12000, 16384]))
        l = int(rng.choice([1, 7, 64, 129, 1000, 2048, 3333, 4096]))
        n = int(rng.choice([1, 65, 128, 700, 1024, 2049, 4096]))
        if m * l * n > 6e10:
            l = max(1, int(6e10 // (m * n)))
        k = int(rng.choice([8, 8, 8, 8, 5, 3]))
        plan = rng.choice(["auto", "auto", "tm", "ws5", "fused", "fusedp"])
        ov = {"auto": (0, 0, -1, 0),
              "tm": (64 if fname == "f2" and rng.random() < 0.5 else TM_RT[fname], int(rng.choice([1, 2, -1])), 6, 256),
              "ws5": (16, -1, 5, 256), "fused": (int(rng.choice([1, 2, 4])), int(rng.choice([1, 4, 16])), 10, 256),
              "fusedp": (int(rng.choice([2, 4])), int(rng.choice([1, 4, 16])), 11, 256)}[plan]
        order = 4 if fname == "gf4" else 8 if fname == "gf8" else p
        A = torch.randint(0, order, (m, l), dtype=torch.uint8, device=dev)
        B = torch.randint(0, order, (l, n), dtype=torch.uint8, device=dev)
        M.set_plan_override(*ov)
        try:
            C = sg.m4rm_multiply(sg.BitslicedMatrix.from_dense(f, A), sg.BitslicedMatrix.from_dense(f, B), sg.M4rmParams(k))
        except RuntimeError as e:
            M.set_plan_override()
            if "no compiled" in str(e):
                continue
            raise
        M.set_plan_override()
        ran += 1
        got = C.to_dense()
        got = torch.as_tensor(np.asarray(got), device=dev)
        want = exact(fname, A, B)
        if not torch.equal(got, want):
            bad += 1
            print("MISMATCH", fname, m, l, n, k, plan, ov, flush=True)
    print(f"parity campaign: {ran} products ({cases} drawn), {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
