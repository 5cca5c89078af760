"""Static SASS statistics of the hot GEMM loop (instructions per MAC, mix).

    python tools/sass_stats.py [kernel-substring]
Counts the instructions of every backward-branch loop that contains IMAD.HI
(FLO: one per posit MAC) in libposit_b200.so, to estimate issue slots per MAC
before spending GPU time.
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.environ.get("POSIT_LIB_PATH", "/root/repo/paper_2401_14117_b200/libposit_b200.so")


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 else "k_gemmILb0ELb0"
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    for f in re.split(r"\n\s+Function : ", txt):
        name = f.split("\n")[0]
        if pat not in name:
            continue
        ins = []
        for l in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        print(name.strip(), "total instructions", len(ins))
        for a, t in ins:
            m = re.search(r"BRA.*?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                tgt = int(m.group(1), 16)
                body = [x[1] for x in ins if tgt <= x[0] <= a]
                nhi = sum(1 for x in body if x.startswith("FLO"))
                if nhi == 0:
                    continue
                print(f"  loop [{tgt:#x},{a:#x}] len {len(body)} products {nhi} -> {len(body) / nhi:.2f} instr/MAC")
                c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
                print("   ", ", ".join(f"{k} {v / nhi:.2f}" for k, v in sorted(c.items(), key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
