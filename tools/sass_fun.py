"""Print the SASS of one kernel from a fatbin/.so: python tools/sass_fun.py LIB REGEX [--hist]"""
import re
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if re.search(pat, name):
        lines = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
        print("==", name, len(lines), "instructions")
        if "--hist" in sys.argv:
            c = Counter(re.sub(r"^\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?", "", l).split()[0].split(".")[0] for l in lines)
            print(c.most_common(25))
        else:
            print("\n".join(l[:110] for l in lines))
