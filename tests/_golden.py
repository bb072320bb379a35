"""Helpers to read the committed golden fixtures (tests/golden, made by make_golden.py)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELD_FILES = {"f2": "m4rm_f2.npz", "f3": "m4rm_f3.npz", "f5": "m4rm_f5.npz", "f7": "m4rm_f7.npz",
               "gf4": "gf4.npz", "z4": "m4rm_z4.npz", "z8": "m4rm_z8.npz"}


def cases(field):
    z = np.load(os.path.join(GOLDEN, FIELD_FILES[field]))
    out = []
    for i in range(int(z["count"])):
        m, l, n, k, sa, sb = (int(x) for x in z[f"c{i}_shape"])
        out.append(dict(m=m, l=l, n=n, k=k, seed_a=sa, seed_b=sb, A=z[f"c{i}_A"], B=z[f"c{i}_B"],
                        C=z[f"c{i}_C"], Craw=z[f"c{i}_Craw"]))
    return out


def kernel_cases():
    with open(os.path.join(GOLDEN, "kernel_cases.json")) as f:
        return json.load(f)
