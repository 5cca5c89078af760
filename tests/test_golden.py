"""The oracle (and, under -m gpu, the CUDA path) against the cited fixtures in
tests/golden/: values fixed by Eq.1, printed by the paper
 or printed as worked examples in SPEC.md."""
import math
from fractions import Fraction

import numpy as np
import pytest

from tests import golden_fixtures as G
from oracle import checker as X
from oracle import oracle as O

ONE, MONE = 0x40000000, 0xC0000000


@pytest.mark.parametrize("pat,val,cite", G.format_constants())
def test_oracle_format_constants(pat, val, cite):
    if val is None:
        assert math.isnan(O.to_f64(pat)) and X.value(pat) is None, cite
        return
    assert Fraction(O.to_f64(pat)) == val, cite
    assert X.value(pat) == val, cite
    assert O.from_f64(float(val)) == pat, cite


@pytest.mark.parametrize("x,fs,cite", G.fraction_bits())
def test_oracle_fraction_bits(x, fs, cite):
    assert O.fraction_bits(O.from_f64(x)) == fs, cite


def _oracle_scalar(op, a, b):
    if op == "f64":
        return O.from_f64(a)
    if op in ("sqrt", "neg"):
        return getattr(O, op)(a)
    return getattr(O, op)(a, b)


@pytest.mark.parametrize("op,a,b,exp,cite", G.spec_scalar())
def test_oracle_spec_scalar(op, a, b, exp, cite):
    assert _oracle_scalar(op, a, b) == exp, cite


@pytest.mark.parametrize("case", G.spec_linalg(), ids=lambda c: c["op"])
def test_oracle_spec_linalg(case):
    P = O.from_f64_array
    if case["op"] == "gemm":
        got = O.gemm(P(case["A"]), P(case["B"]), np.zeros((2, 2), np.uint32), alpha=ONE, beta=0)
        assert np.array_equal(got, P(case["expect"]))
    elif case["op"] == "getrf":
        lu, ipiv, info = O.getrf(P(case["A"]))
        assert np.array_equal(np.triu(O.to_f64_array(lu)), case["expect"])
        assert list(ipiv) == case["ipiv"] and info == case["info"]
        assert np.all(np.tril(O.to_f64_array(lu), -1) == 0)        # L21 = 0
    elif case["op"] == "potrf":
        l, info = O.potrf_lower(P(case["A"]))
        assert np.array_equal(np.tril(O.to_f64_array(l)), case["expect"]) and info == case["info"]
    elif case["op"] == "trsm_rltn":
        got = O.trsm_rltn(P(case["L"]), P(case["B"]))
        assert np.array_equal(O.to_f64_array(got), case["expect"])
    elif case["op"] == "potrs":
        l, info = O.potrf_lower(P(case["A"]))
        assert np.array_equal(O.to_f64_array(O.potrs_lower(l, P(case["b"]))), case["expect"])


# ---- the CUDA path against the same fixtures (values, not the oracle) --------
@pytest.mark.gpu
def test_gpu_golden_scalar_and_constants(cuda_ok):
    import torch
    import paper_2401_14117_b200 as PB
    from tests.gpu_util import to_dev, to_host
    for op, a, b, exp, cite in G.spec_scalar():
        if op == "f64":
            got = to_host(PB.posit_from_f64(torch.tensor([a], dtype=torch.float64, device="cuda")))[0]
        elif op == "neg":
            got = to_host(PB.posit_vec_op("sub", to_dev(np.array([0], np.uint32)), to_dev(np.array([a], np.uint32))))[0]
        else:
            bb = np.array([a if b is None else b], np.uint32)
            got = to_host(PB.posit_vec_op(op, to_dev(np.array([a], np.uint32)), to_dev(bb)))[0]
        assert int(got) == exp, (op, cite)
    for pat, val, cite in G.format_constants():
        got = PB.posit_to_f64(to_dev(np.array([pat], np.uint32))).cpu().numpy()[0]
        assert (math.isnan(got) if val is None else Fraction(float(got)) == val), cite


@pytest.mark.gpu
def test_gpu_golden_linalg(cuda_ok):
    import torch
    import paper_2401_14117_b200 as PB
    from tests.gpu_util import to_host

    def dev(x):
        return PB.posit_from_f64(torch.tensor(x, dtype=torch.float64, device="cuda"))

    def f64(t):
        return PB.posit_to_f64(t).cpu().numpy()

    for case in G.spec_linalg():
        if case["op"] == "gemm":
            C = dev(np.zeros((2, 2)))
            PB.posit_gemm(dev(case["A"]), dev(case["B"]), C, alpha=ONE, beta=0)
            assert np.array_equal(f64(C), case["expect"])
        elif case["op"] == "getrf":
            A = dev(case["A"])
            ipiv = torch.zeros(2, dtype=torch.int32, device="cuda")
            info = torch.zeros(1, dtype=torch.int32, device="cuda")
            PB.posit_getrf(A, ipiv, info, nb=1)
            assert np.array_equal(np.triu(f64(A)), case["expect"]) and np.all(np.tril(f64(A), -1) == 0)
            assert ipiv.cpu().tolist() == case["ipiv"] and int(info.cpu()[0]) == case["info"]
        elif case["op"] == "potrf":
            A = dev(case["A"])
            info = torch.zeros(1, dtype=torch.int32, device="cuda")
            PB.posit_potrf(A, info, nb=1)
            assert np.array_equal(np.tril(f64(A)), case["expect"]) and int(info.cpu()[0]) == case["info"]
        elif case["op"] == "trsm_rltn":
            B = dev(case["B"])
            PB.posit_trsm("R", "L", "T", "N", dev(case["L"]), B)
            assert np.array_equal(f64(B), case["expect"])
        elif case["op"] == "potrs":
            A = dev(case["A"])
            info = torch.zeros(1, dtype=torch.int32, device="cuda")
            PB.posit_potrf(A, info, nb=1)
            b = dev(case["b"])
            PB.posit_potrs(A, b)
            assert np.array_equal(f64(b), case["expect"])
        to_host(torch.zeros(1, device="cuda"))
