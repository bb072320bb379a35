import sys
# mod-15 (4-bit value 0..15) -> canonical F5 residue (3 bits)
pts = [(v, v % 5) for v in range(16)]
print(4, 3, len(pts))
for a, b in pts: print(a, b)
