"""Plan multi-operand carry-save accumulation modulo 2^n - 1 with LOP3 full/half adders.

State: bits per column (column i has weight 2^i; a carry out of column n-1 re-enters column 0,
since 2^n == 1 mod 2^n - 1).  FA: 3 bits of a column -> 1 sum bit (same column) + 1 carry
(next column), 2 LOP3.  HA: 2 bits -> 1 + 1 carry, 2 LOP3.  Find the cheapest sequence that
brings the per-column counts under `cap` (the accumulator's planes per column).
"""
import heapq
import itertools
import sys


def plan(counts, cap, max_cost=40):
    n = len(counts)
    start = tuple(counts)
    pq = [(0, start, ())]
    seen = {start: 0}
    while pq:
        cost, st, ops = heapq.heappop(pq)
        if all(st[i] <= cap[i] for i in range(n)):
            return cost, ops
        if cost >= max_cost:
            continue
        for i in range(n):
            for kind, need in (("FA", 3), ("HA", 2)):
                if st[i] >= need:
                    nx = list(st)
                    nx[i] -= need - 1
                    nx[(i + 1) % n] += 1
                    nx = tuple(nx)
                    c = cost + 2
                    if seen.get(nx, 1 << 30) > c:
                        seen[nx] = c
                        heapq.heappush(pq, (c, nx, ops + ((kind, i),)))
    return None


if __name__ == "__main__":
    # F7: state caps per column + inputs x (0,1,2), 2y (1,2,0), 4z (2,0,1)
    for cap in [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]:
        counts = [cap[i] + 3 for i in range(3)]
        print("F7 cap", cap, "->", plan(counts, cap))
    # F5 mod 15: inputs x (0,1,2), 2y (1,2,3), 4z (2,3,0)  -> per column (2,2,3,2)
    # or with -z instead of 4z: (2,3,3,1)
    for name, inp in (("4z", (2, 2, 3, 2)), ("-z", (2, 3, 3, 1))):
        for cap in itertools.product((1, 2), repeat=4):
            counts = [cap[i] + inp[i] for i in range(4)]
            r = plan(counts, cap)
            if r:
                print("F5", name, "cap", cap, "planes", sum(cap), "-> LOP3", r[0], r[1])
