"""Per-instruction view of an ncu `--page source --csv --print-source sass` export: shared-memory
wavefronts by opcode, and the hottest instructions by stall samples.

python tools/ncu_sass_hot.py gpurun_out/X_sass.csv [top]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(j for j, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[i]
    return [dict(zip(hdr, r)) for r in rows[i + 1:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, top=40):
    rs = load(path)
    wf = collections.Counter()
    ideal = collections.Counter()
    ex = collections.Counter()
    samples = collections.Counter()
    tot_s = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rs)
    for r in rs:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        wf[op] += num(r["L1 Wavefronts Shared"])
        ideal[op] += num(r["L1 Wavefronts Shared Ideal"])
        ex[op] += num(r["Instructions Executed"])
        samples[op.split(".")[0]] += num(r["Warp Stall Sampling (All Samples)"])
    tw = sum(wf.values())
    print(f"shared wavefronts {tw:.4g}")
    for op, v in wf.most_common(12):
        if v:
            print(f"  {op:28s} {v:12.4g} ({100 * v / tw:5.1f} %)  ideal {ideal[op]:.4g}  executed {ex[op]:.4g}")
    print("stall samples by opcode:")
    for op, v in samples.most_common(15):
        print(f"  {op:12s} {100 * v / tot_s:5.1f} %")
    stall_cols = [k for k in rs[0] if k.startswith("stall_") and "Not Issued" not in k]
    print(f"top {top} instructions by samples:")
    for r in sorted(rs, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]:
        st = sorted(((num(r[k]), k[6:]) for k in stall_cols), reverse=True)[:3]
        print(f"  {r['Address'][-5:]} {100 * num(r['Warp Stall Sampling (All Samples)']) / tot_s:5.2f}%  "
              f"{r['Source'].strip()[:60]:60s} " + " ".join(f"{n}={int(v)}" for v, n in st if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
