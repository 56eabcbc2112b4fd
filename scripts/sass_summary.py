"""SASS opcode summary of chosen kernels in libdictmerge.so (run here, no GPU):
opcode histogram, and the Blackwell features the kernels use (UBLKCP = TMA bulk
copy, SYNCS = mbarrier transactions), registers / spills from the cubin.

    python scripts/sass_summary.py 'k_recompressILi24ELi2E' 'k_sp_write' ..."""
import collections
import re
import subprocess
import sys

LIB = "paper_1109_6885_b200/libdictmerge.so"
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for pat in sys.argv[1:] or ["k_recompressILi24ELi2E"]:
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if pat not in name:
            continue
        ops = collections.Counter()
        for m in re.finditer(r"/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", f):
            ops[m.group(1)] += 1
        total = sum(ops.values())
        print(f"== {name}")
        print(f"   static instructions: {total}")
        print("   " + " ".join(f"{k}:{v}" for k, v in ops.most_common(40)))
        feats = {k: ops.get(k, 0) for k in ("UBLKCP", "SYNCS", "UTMALDG", "UTMASTG", "LDS", "STS", "SHFL", "LDG", "STG",
                                           "POPC", "ATOMS", "ATOMG", "RED")}
        print("   features: " + " ".join(f"{k}={v}" for k, v in feats.items()))
        break
