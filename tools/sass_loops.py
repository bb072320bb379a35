"""Loops of one kernel's SASS: backward branches, their size and opcode histogram.
python tools/sass_loops.py OBJ REGEX"""
import re
import subprocess
import sys
from collections import Counter


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s+Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        ins = []
        for l in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        yield name, ins


def opcode(text):
    t = re.sub(r"^@!?U?P\w+\s+", "", text)
    return t.split()[0]


def loops(ins):
    """[(start_addr, end_addr)] of backward branches (innermost first by size)."""
    out = []
    for addr, text in ins:
        op = opcode(text)
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", text.split(" ", 1)[1] if " " in text else "")
            if m:
                tgt = int(m.group(1), 16)
                if tgt <= addr:
                    out.append((tgt, addr))
    return sorted(out, key=lambda x: x[1] - x[0])


if __name__ == "__main__":
    for name, ins in functions(sys.argv[1]):
        if not re.search(sys.argv[2], name):
            continue
        print("==", name, len(ins))
        for a, b in loops(ins):
            body = [t for x, t in ins if a <= x <= b]
            c = Counter(opcode(t).split(".")[0] for t in body)
            print(f"  loop {a:#x}-{b:#x}: {len(body)} instr", c.most_common(12))
