"""Per-kernel SASS instruction counts of libgc3.so (cuobjdump -sass): the evidence that the
interpreter uses the Blackwell bulk-copy engine (UBLKCP = cp.async.bulk, UBLKRED =
cp.reduce.async.bulk), mbarriers (SYNCS.*) and 128-bit global accesses.

    python tools/sass_counts.py [libgc3.so] [--sass dump.txt] > profiles/<tag>_sass_counts.md
"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

KEYS = ["UBLKCP", "UBLKRED", "SYNCS", "LDG.E.128", "STG.E.128", "LDG.E.ENL2.128", "ERRBAR", "MEMBAR", "BAR.RED", "BAR.SYNC",
        "B2R.RESULT", "ATOMG", "RED.E", "CCTL"]


def demangle(names):
    p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return p.stdout.split("\n")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    lib = args[0] if args else "paper_2201_11840_b200/libgc3.so"
    if "--sass" in sys.argv:
        text = open(sys.argv[sys.argv.index("--sass") + 1]).read()
    else:
        text = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = OrderedDict()
    cur = None
    for line in text.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        funcs[cur]["_total"] += 1
        for k in KEYS:
            if op.startswith(k):
                funcs[cur][k] += 1
    names = demangle(list(funcs))
    print("# SASS instruction counts per kernel (`cuobjdump -sass " + lib + "`, sm_100a)\n")
    print("UBLKCP = `cp.async.bulk` (bulk copy engine), UBLKRED = `cp.reduce.async.bulk` (L2 reduction), "
          "SYNCS = mbarrier ops, B2R.RESULT = `bar.red` result.\n")
    print("| kernel | instr | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    tot = Counter()
    for (mangled, c), name in zip(funcs.items(), names):
        tot.update(c)
        short = name.replace("gc3::dev::", "").replace("(gc3::LaunchArgs)", "").replace("gc3::", "")
        print(f"| `{short}` | {c['_total']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")
    print(f"| **all {len(funcs)} kernels** | {tot['_total']} | " + " | ".join(str(tot[k]) for k in KEYS) + " |")


if __name__ == "__main__":
    main()
