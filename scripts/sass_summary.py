"""Per-kernel SASS evidence of liblsw.so (cuobjdump -sass): counts of the
Blackwell instructions that show what each kernel runs on -- tcgen05 MMA
(UTCHMMA / UTCQMMA), commits (UTCBAR), TMEM loads (LDTM), TMA tensor loads /
stores (UTMALDG / UTMASTG), bulk copies (UBLKCP), mbarrier waits
(SYNCS.PHASECHK), packed fp32 math (FFMA2 / FADD2), shuffles -- plus a short
excerpt around the first MMA.  Writes Markdown to stdout."""
import os
import re
import subprocess
import sys
from collections import Counter, OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2405_17741_b200", "liblsw.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "SYNCS.PHASECHK",
        "SYNCS.ARRIVE", "FFMA2", "FADD2", "FFMA", "SHFL", "RED", "ATOM", "DMUL", "DFMA", "F2FP.BF16"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            funcs[cur].append(ln.strip())
    dem = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
    print("# SASS evidence: liblsw.so (sm_100a)\n")
    print("`cuobjdump -sass paper_2405_17741_b200/liblsw.so`, counted by `scripts/sass_summary.py`.\n")
    print("| kernel | instr | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    excerpts = []
    for (name, lines), nice in zip(funcs.items(), dem):
        ops = Counter()
        for l in lines:
            body = re.sub(r"^/\*[0-9a-f]{4,}\*/\s*", "", l)
            body = re.sub(r"^@!?U?P\w+\s+", "", body)
            op = body.split()[0] if body else ""
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    ops[k] += 1
        short = re.sub(r"\(.*", "", nice).replace("lsw::", "")
        print(f"| `{short}` | {len(lines)} | " + " | ".join(str(ops[k]) if ops[k] else "" for k in KEYS) + " |")
        first = next((i for i, l in enumerate(lines) if "UTCHMMA" in l), None)
        if first is not None:
            excerpts.append((short, lines[max(0, first - 6): first + 6]))
    print("\n## Excerpts (around the first tcgen05 MMA of each kernel)\n")
    for short, ex in excerpts:
        print(f"`{short}`\n```")
        print("\n".join(ex))
        print("```\n")


if __name__ == "__main__":
    main()
