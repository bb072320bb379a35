"""Per-(row, k-block) instruction mix of every k = 8 M4RM instantiation, counted from the compiled
SASS (cuobjdump of csrc/build/sg_m4rm_<field>.o).

The lookup warps' main loop (the smallest backward-branch loop that issues at least RT * NI * R
LDS and no STS -- the table stores belong to the builder warps) is one k-block for RT row-slots;
its opcode counts / RT are the instructions one lane spends per (row, k-block, 128-column slab).
bench.py turns them into the integer-pipe roofline.  Writes
profiles/<tag>_sass_mix.json.   python tools/sass_mix.py r02"""
import json
import os
import re
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_loops import functions, loops, opcode  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_0901_1413_b200", "csrc", "build")
FIELDS = {0: ("f2", 1, 1), 1: ("f3", 2, 2), 2: ("f5", 3, 3), 3: ("f7", 3, 3), 4: ("gf4", 2, 2), 5: ("gf8", 3, 3),
          6: ("z4", 2, 2), 7: ("z8", 3, 3)}  # code -> (name, R, NI)
# integer (ALU) pipe vs FMA pipe vs shared memory, as nvdisasm opcodes
ALU = {"LOP3", "PRMT", "LEA", "SHF", "IADD3", "ISETP", "SEL", "PLOP3", "LOP", "MOV", "IABS", "FLO", "POPC", "BMSK"}
FMA = {"IMAD", "VIADD", "IMNMX", "VIMNMX", "IMUL"}


def mix_of(fname, ins, field_code, rt, sched, nt):
    name, R, NI = FIELDS[field_code]
    best = None
    for a, b in loops(ins):
        body = [t for x, t in ins if a <= x <= b]
        c = Counter(opcode(t).split(".")[0] for t in body)
        # the lookup loop: RT row-slots of NI x R table loads, with the field arithmetic; in the
        # warp-specialized schedule it holds no table stores (those are the builder warps')
        # (GF(4), k = 8: Karatsuba tables, three one-plane lookups per row)
        nl = 3 if name == "gf4" else NI * R
        if c["LDS"] >= rt * nl and c["LOP3"] >= rt and (sched not in (2, 5, 6) or c["STS"] == 0):
            best = (a, b, c)
            break  # loops() is sorted by size: the smallest qualifying loop
    if best is None:
        return None
    a, b, c = best
    per = {k: v / rt for k, v in sorted(c.items())}
    return {"field": name, "rt": rt, "sched": sched, "threads": nt, "loop": [hex(a), hex(b)],
            "loop_instructions": sum(c.values()),
            "includes_table_build": sched not in (2, 5, 6),
            "per_row_block": per,
            "alu_per_row_block": sum(v for k, v in per.items() if k in ALU),
            "lop3_per_row_block": per.get("LOP3", 0.0),
            "fma_per_row_block": sum(v for k, v in per.items() if k in FMA),
            "lds_per_row_block": per.get("LDS", 0.0),
            "issue_per_row_block": sum(per.values())}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = {"_source": "tools/sass_mix.py: cuobjdump -sass of csrc/build/*.o, lookup loop / RT",
           "_alu_opcodes": sorted(ALU), "_fma_opcodes": sorted(FMA)}
    for code, (name, R, NI) in FIELDS.items():
        obj = os.path.join(BUILD, f"sg_m4rm_{name}.o")
        if not os.path.exists(obj):
            continue
        for fname, ins in functions(obj):
            # the resident-B, unfused instantiations (STRM = FUSED = false)
            m = re.search(rf"m4rm_kernelILi{code}ELi8ELi(\d+)ELi(\d)ELi(\d+)ELi0ELb0ELb0E", fname)
            if not m:
                continue
            rt, sched, nt = (int(x) for x in m.groups())
            if sched == 6:  # second accumulator set in TMEM: the loop covers 2 RT row-slots
                rt *= 2
            mix = mix_of(fname, ins, code, rt, sched, nt)
            if mix:
                out[f"{name}/{rt}/{sched}/{nt}"] = mix
    path = os.path.join(ROOT, "profiles", f"{tag}_sass_mix.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    for k, v in out.items():
        if not k.startswith("_"):
            print(k, "alu %.1f lop3 %.1f fma %.1f lds %.1f issue %.1f" % (
                v["alu_per_row_block"], v["lop3_per_row_block"], v["fma_per_row_block"], v["lds_per_row_block"],
                v["issue_per_row_block"]))


if __name__ == "__main__":
    main()
