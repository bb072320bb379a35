import sys; sys.path.insert(0, '.')
import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import m4rm as M, _lib
import ctypes
L = _lib.load()
for args in ((16, 1, 3, 224), (16, 0, 3, 0), (0, 0, 3, 0)):
    M.set_plan_override(*args)
    try:
        print(args, sg.plan(sg.F3, 32768, 32768, 32768, 8))
    except Exception as e:
        print(args, "ERR", e)
