"""Flip compiled-in defaults after an A/B (edits the sources; rebuild afterwards).
    python tools/flip_defaults.py [potf2_ddiv=1] [leaf_ddiv=1] [pc_packed=1] [bk=32] [potf2_defer=1]"""
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
C = os.path.join(ROOT, "paper_2401_14117_b200", "csrc")


def sub(path, pat, rep, count=1):
    s = open(path).read()
    s2, n = re.subn(pat, rep, s, count=count, flags=re.S)
    assert n == count, (path, pat, n)
    open(path, "w").write(s2)


for a in sys.argv[1:]:
    k, v = a.split("=")
    if k == "potf2_ddiv":
        sub(os.path.join(C, "chol.cu"), r'(getenv\("POSIT_POTF2_DDIV"\);\s*return e \? atoi\(e\) != 0 : )(true|false);[^\n]*',
            r"\g<1>" + ("true" if v == "1" else "false") + ";   // measured: see DESIGN.md section 8")
    elif k == "leaf_ddiv":
        sub(os.path.join(C, "leaf.cu"), r'(getenv\("POSIT_LEAF_DDIV"\);\s*return e \? atoi\(e\) : )[01];[^\n]*',
            r"\g<1>" + v + ";   // measured: see DESIGN.md section 8")
    elif k == "leaf_rows":
        sub(os.path.join(C, "leaf.cu"), r'(getenv\("POSIT_LEAF_ROWS"\);\s*return e \? atoi\(e\) : )[01];[^\n]*',
            r"\g<1>" + v + ";   // measured: see DESIGN.md section 8")
    elif k == "wide_leaf_cols":
        sub(os.path.join(C, "capi.cu"), r'(getenv\("POSIT_WIDE_LEAF_COLS"\);\s*return e \? \(int64_t\)atoll\(e\) : \(int64_t\))\d+;',
            r"\g<1>" + v + ";")
    elif k == "side_min":
        sub(os.path.join(C, "leaf.cu"), r"const int64_t side_auto = \(m \+ 1023\) / 1024 < \d+ \? \d+ :",
            f"const int64_t side_auto = (m + 1023) / 1024 < {v} ? {v} :")
    elif k == "pc_packed":
        sub(os.path.join(C, "chol.cu"), r"#define PC_PACKED [01]", f"#define PC_PACKED {v}")
    elif k == "bk":
        sub(os.path.join(C, "gemm_d.cu"), r"#define PGD_BK \d+ ", f"#define PGD_BK {v} ")
    elif k == "potf2_defer":
        sub(os.path.join(C, "chol.cu"), r'(getenv\("POSIT_POTF2_DEFER"\);\s*return \(e && atoi\(e\) == 1\) \? 1 : )0;',
            r"\g<1>0;" if v == "0" else r"\g<1>0;")
    else:
        raise SystemExit(f"unknown key {k}")
    print("set", k, v)
