"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/*.h declares, and its host-side contract checks raise the
reference's exception types with the reference's messages -- all without a
GPU (no compute call is made)."""
import inspect

import numpy as np
import pytest

import paper_1303_4312_b200 as P
from paper_1303_4312_b200 import _native as N


def test_library_exports_every_declared_symbol():
    names = N.declared_symbols()
    assert len(names) >= 30
    missing = [s for s in names if not hasattr(N.lib, s)]
    assert not missing, missing
    assert N.lib.comerge_cuda_abi_version() == 10000
    # the product exports no test infrastructure
    assert not any(hasattr(N.lib, s) for s in N.declared_symbols(N.TESTKIT_HEADERS))


def test_testkit_library_is_separate_and_complete():
    names = N.declared_symbols(N.TESTKIT_HEADERS)
    assert names and all(n.startswith("comerge_testkit_") for n in names)
    missing = [s for s in names if not hasattr(N.tk(), s)]
    assert not missing, missing


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_partition_output_kats(kat):
    for case in kat["partition_output"]:
        if "expect" in case:
            assert [P.partition_output(case["total"], case["workers"], r)
                    for r in range(case["workers"] + 1)] == case["expect"], case["src"]
        else:
            assert P.partition_output(case["total"], case["workers"], case["r"]) == case["expect_r"]
    for case in kat["partition_output_errors"]:
        with pytest.raises(ValueError):
            P.partition_output(case["total"], case["workers"], case["r"])


def test_partition_output_balance():
    """parallel_test.cpp:46-62: block sizes never differ by more than one."""
    for total in range(0, 120):
        for p in range(1, 18):
            sizes = [P.partition_output(total, p, r + 1) - P.partition_output(total, p, r)
                     for r in range(p)]
            assert sum(sizes) == total
            assert max(sizes) - min(sizes) <= 1


def test_co_rank_out_of_range_message(kat):
    for case in kat["co_rank_errors"]:
        with pytest.raises(IndexError, match=case["message"]):
            P.co_rank(case["i"], np.array(case["a"], np.uint64), np.array(case["b"], np.uint64))


def test_merge_parallel_contract_errors(kat):
    for case in kat["merge_parallel_errors"]:
        a, b = np.array(case["a"], np.uint64), np.array(case["b"], np.uint64)
        out = np.zeros(case["out_len"], np.uint64)
        with pytest.raises(ValueError, match=case["message"]):
            P.merge_parallel(a, b, out, case["workers"])


def test_merge_errors(kat):
    for case in kat["merge_errors"]:
        a, b = np.array(case["a"], np.uint64), np.array(case["b"], np.uint64)
        with pytest.raises(ValueError, match=case["message"]):
            P.stable_merge(a, b, np.zeros(case["out_len"], np.uint64))


def test_alias_rejected_before_any_device_work():
    buf = np.array([1, 2, 3, 0, 0, 0], np.uint64)   # merge_test.cpp:61-66
    with pytest.raises(ValueError, match="must not alias"):
        P.merge_parallel(buf[0:2], buf[2:3], buf[1:4], 2)


def test_length_error():
    """check_total_length (corank.hpp:67-70) -> OverflowError."""
    import ctypes as C
    rc = N.lib.comerge_merge_parallel_u64(None, 2**63, None, 2**63 + 5, None, 0, 1, 0, None, None,
                                          None)
    assert rc == N.E_LENGTH and "exceeds index range" in N.last_error()
    j, k = C.c_uint64(), C.c_uint64()
    rc = N.lib.comerge_co_rank_u64(0, None, 2**64 - 1, None, 2, C.byref(j), C.byref(k), None, None)
    assert rc == N.E_LENGTH


def test_python_mirror_names_follow_reference():
    for name in ("co_rank", "co_rank_counted", "stable_merge", "partition_output", "plan",
                 "merge_parallel", "merge_parallel_synced"):
        assert callable(getattr(P, name))
    sig = inspect.signature(P.merge_parallel)
    assert list(sig.parameters)[:4] == ["a", "b", "out", "workers"]
    rep = P.MergeReport()
    for f in ("m", "n", "workers", "wall_ns", "block_sizes", "corank_iterations", "comparisons",
              "verified", "speedup_vs_p1", "note"):
        assert hasattr(rep, f)


def test_custom_ordering_rejected():
    with pytest.raises(TypeError):
        P.merge_parallel(np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(2, np.uint64), 1,
                         less=lambda x, y: x > y)
