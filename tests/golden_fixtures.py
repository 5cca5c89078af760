"""Readers for the cited fixtures under tests/golden/ (values printed by the
paper / SPEC or fixed by Eq.1; each line carries its citation)."""
import os
from fractions import Fraction

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def _exact(tok):
    """'0', '1/2', '2^-27', '1+2^-27', '-1' -> Fraction; 'NaR' -> None."""
    if tok == "NaR":
        return None
    if "+" in tok:
        a, b = tok.split("+", 1)
        return _exact(a) + _exact(b)
    if tok.startswith("-"):
        return -_exact(tok[1:])
    if "^" in tok:
        base, ex = tok.split("^")
        return Fraction(int(base)) ** int(ex)
    return Fraction(tok)


def format_constants():
    out = []
    for line in _lines("format_constants.txt"):
        pat, val, cite = line.split(None, 2)
        out.append((int(pat, 16), _exact(val), cite))
    return out


def spec_scalar():
    out = []
    for line in _lines("spec_scalar.txt"):
        op, a, b, exp, cite = line.split(None, 4)
        a = float(a) if op == "f64" else int(a, 16)
        b = None if b == "-" else int(b, 16)
        out.append((op, a, b, int(exp, 16), cite))
    return out


def fraction_bits():
    return [(float(v), int(f), c) for v, f, c in (l.split(None, 2) for l in _lines("fraction_bits.txt"))]


def _mat(s):
    return np.array([[float(x) for x in row.split(",")] for row in s.split(";")])


def spec_linalg():
    out = []
    for line in _lines("spec_linalg.txt"):
        toks = line.split()
        case = {"op": toks[0]}
        for t in toks[1:]:
            k, v = t.split("=")
            if k == "ipiv":
                case[k] = [int(x) for x in v.split(",")]
            elif k == "info":
                case[k] = int(v)
            elif k == "b" or (case["op"] == "potrs" and k == "expect"):
                case[k] = np.array([float(x) for x in v.split(",")])
            else:
                case[k] = _mat(v)
        out.append(case)
    return out
