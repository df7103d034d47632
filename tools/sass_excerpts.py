"""Key SASS instructions per kernel of the built library (profiles/r02_sass_excerpts.txt).

    python tools/sass_excerpts.py > profiles/r02_sass_excerpts.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_1811_07717_b200/_lib/libhfb200.so"
KERNELS = ["_ZN2hf3pcg10k_update_rILi64EEEvNS0_3CtlEPKdPd",
           "_ZN2hf3pcg6k_spmmILi64ELi0EEEvNS0_3CtlENS0_3EllEPKdS5_Pd",
           "_ZN2hf3pcg6k_spmmILi32ELi0EEEvNS0_3CtlENS0_3EllEPKdS5_Pd",
           "_ZN2hf3pcg10k_update_pILi64EEEvNS0_3CtlEPKdPdS4_",
           "k_lf_tile", "k_eit_sens"]
KEY = re.compile(r"(ENL2\.256|DMMA)")


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    print(f"# cuobjdump -sass {LIB} (sm_100a): key instructions per kernel")
    print("# LDG.E.ENL2.256 / STG.E.ENL2.256 = 256-bit global accesses (4 fp64 per lane, kp = 32 and 64);")
    print("# DMMA.8x8x4 = the fp64 tensor-core mma.sync.m8n8k4 (tcgen05 has no fp64 kind)")
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not any(k == name or (k in name and not k.startswith("_Z")) for k in KERNELS):
            continue
        lines = [ln for ln in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4}\*/", ln)]
        ops = collections.Counter()
        for ln in lines:
            m = re.search(r"\*/\s+(@!?P\d\s+)?([A-Z][A-Z0-9]*)", ln)
            if m:
                ops[m.group(2)] += 1
        print(f"\n== {name}")
        print("   counts:", {k: ops[k] for k in ("LDG", "STG", "LDS", "DFMA", "DMMA") if ops[k]})
        shown = 0
        for ln in lines:
            if KEY.search(ln) and shown < 6:
                print("  ", ln.strip())
                shown += 1


if __name__ == "__main__":
    sys.exit(main())
