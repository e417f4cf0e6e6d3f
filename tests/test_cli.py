"""The B200 command line tool (bin/comerge_cuda, cli/) against the reference
CLI's own end-to-end cases (proj/tests/cli_test.cpp) and the reference's
bench numbers (tests/golden section 9).

Error paths that never reach the device run without a GPU; everything that
merges or co-ranks is marked gpu."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "bin", "comerge_cuda")

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="bin/comerge_cuda not built")


def run(*args):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


def text_file(path, keys):
    with open(path, "w") as f:
        for k in keys:
            f.write(f"{k}\n")
    return str(path)


def crmg_file(path, keys, version=1, count=None):
    """CRMG binary: magic | version u8 | flags u8 | count u64 LE | keys u64 LE (io.hpp:11-20)"""
    keys = list(keys)
    with open(path, "wb") as f:
        f.write(b"CRMG" + bytes([version, 0]) + struct.pack("<Q", len(keys) if count is None else count))
        f.write(b"".join(struct.pack("<Q", k) for k in keys))
    return str(path)


def read_crmg(path):
    data = open(path, "rb").read()
    assert data[:4] == b"CRMG" and data[4] == 1
    (count,) = struct.unpack("<Q", data[6:14])
    return list(struct.unpack(f"<{count}Q", data[14:14 + 8 * count]))


# ------------------------------------------------- no device needed

def test_exit_codes_usage_and_io(tmp_path):
    """cli_test.cpp:226-241 (the paths that fail before any device work)."""
    a = text_file(tmp_path / "a.txt", [1, 2])
    assert run("frobnicate")[0] == 2                       # unknown command
    assert run("corank", a)[0] == 2                        # missing args
    assert run("corank", a, tmp_path / "nope", 1)[0] == 3  # missing file
    u = text_file(tmp_path / "u.txt", [2, 1])
    assert run("corank", a, u, 1)[0] == 2                  # unsorted input
    assert run("bench", "--dist", "zipf")[0] == 2          # unknown distribution
    assert run("bench", "--dist", "uniform:3")[0] == 2     # takes no parameter
    assert run("bench", "--p-list", "1,0")[0] == 2
    assert run("merge", a, a, tmp_path / "o", "--format", "csv")[0] in (2,)
    code, out, _ = run("--help")
    assert code == 0 and "corank" in out


def test_key_file_errors(tmp_path):
    """io.cpp:59-75: truncated header, bad version, count mismatch, bad text."""
    a = text_file(tmp_path / "a.txt", [1, 2])
    bad = tmp_path / "t.bin"
    bad.write_bytes(b"CRMG\x01")
    assert run("corank", a, bad, 0)[0] == 3
    assert run("corank", a, crmg_file(tmp_path / "v.bin", [1], version=2), 0)[0] == 3
    assert run("corank", a, crmg_file(tmp_path / "c.bin", [1, 2], count=3), 0)[0] == 3
    t = tmp_path / "x.txt"
    t.write_text("1\nseven\n")
    code, _, err = run("corank", a, t, 0)
    assert code == 3 and "x.txt:2" in err


def test_verify_length_mismatch_text_and_binary(tmp_path):
    """cli_test.cpp:103-108: wrong length is reported as such (no device work)."""
    a = text_file(tmp_path / "a.txt", [1, 2, 10, 10])
    b = text_file(tmp_path / "b.txt", [3, 10, 11])
    m = text_file(tmp_path / "m.txt", [1, 2, 3, 10, 10, 10])
    code, _, err = run("verify", a, b, m)
    assert code == 1 and "length mismatch" in err
    ab = crmg_file(tmp_path / "a.bin", [1, 5])
    bb = crmg_file(tmp_path / "b.bin", [2, 4])
    mb = crmg_file(tmp_path / "m.bin", [1, 2, 4])
    code, _, err = run("verify", ab, bb, mb)
    assert code == 1 and "expected 4 keys, found 3" in err


# ------------------------------------------------------ on the device

@pytest.mark.gpu
def test_corank_prints_split_and_cost(tmp_path):
    """cli_test.cpp:69-85."""
    a = text_file(tmp_path / "a.txt", [1, 3, 5, 7])
    b = text_file(tmp_path / "b.txt", [2, 4, 6, 8])
    code, out, _ = run("corank", a, b, 4)
    assert code == 0 and out.startswith("2 2 ")
    assert run("corank", a, b, 0)[1] == "0 0 0 0\n"
    code, _, err = run("corank", a, b, 9)
    assert code == 2 and "rank out of range" in err
    u = text_file(tmp_path / "u.txt", [2, 1])
    assert run("corank", a, u, 1, "--no-validate")[0] == 0


@pytest.mark.gpu
def test_merge_then_verify(tmp_path):
    """cli_test.cpp:87-109."""
    a = text_file(tmp_path / "a.txt", [1, 2, 10, 10])
    b = text_file(tmp_path / "b.txt", [3, 10, 11])
    out = tmp_path / "out.txt"
    code, stdout, _ = run("merge", a, b, out, "--threads", 3)
    assert code == 0 and out.read_text() == "1\n2\n3\n10\n10\n10\n11\n"
    assert stdout.startswith("merged 4 + 3 keys with 3 workers in ")
    assert run("verify", a, b, out)[0] == 0
    text_file(out, [1, 3, 2, 10, 10, 10, 11])
    assert run("verify", a, b, out)[0] == 1


@pytest.mark.gpu
def test_disjoint_empty_and_thread_independence(tmp_path):
    """cli_test.cpp:111-156."""
    a = text_file(tmp_path / "a.txt", [1, 2, 3])
    b = text_file(tmp_path / "b.txt", [10, 20])
    out = tmp_path / "o.txt"
    assert run("merge", a, b, out)[0] == 0 and out.read_text() == "1\n2\n3\n10\n20\n"
    e = text_file(tmp_path / "e.txt", [])
    b2 = text_file(tmp_path / "b2.txt", [4, 5, 6])
    assert run("merge", e, b2, out)[0] == 0 and out.read_text() == open(b2).read()
    ka = [3 * t // 2 for t in range(5000)]
    kb = [t + 1000 for t in range(5000)]
    fa, fb = text_file(tmp_path / "ka.txt", ka), text_file(tmp_path / "kb.txt", kb)
    one, eight = tmp_path / "one.txt", tmp_path / "eight.txt"
    assert run("merge", fa, fb, one, "--threads", 1)[0] == 0
    assert run("merge", fa, fb, eight, "--threads", 8)[0] == 0
    assert one.read_text() == eight.read_text()
    assert [int(x) for x in one.read_text().split()] == sorted(ka + kb)


@pytest.mark.gpu
def test_binary_in_binary_out(tmp_path):
    """cli_test.cpp:158-171, plus --format conversions."""
    a = crmg_file(tmp_path / "a.bin", [1, 5])
    b = crmg_file(tmp_path / "b.bin", [2, 4])
    out = tmp_path / "out.bin"
    assert run("merge", a, b, out)[0] == 0
    assert read_crmg(out) == [1, 2, 4, 5]
    txt = tmp_path / "out.txt"
    assert run("merge", a, b, txt, "--format", "text")[0] == 0
    assert txt.read_text() == "1\n2\n4\n5\n"
    big = [2**64 - 1 - k for k in range(3)][::-1]  # full 64-bit range survives
    fb = crmg_file(tmp_path / "big.bin", big)
    assert run("merge", fb, crmg_file(tmp_path / "z.bin", [0]), out)[0] == 0
    assert read_crmg(out) == [0] + big


@pytest.mark.gpu
def test_bench_csv_matches_reference_counts(tmp_path, golden):
    """cli_test.cpp:173-224, and the comparison counts are the reference's own
    (tests/golden section 9) for every distribution."""
    for token in ("uniform", "all-equal", "few-distinct:16", "disjoint", "interleaved",
                  "organ-pipe", "runs:32"):
        csv = tmp_path / "r.csv"
        code, _, err = run("bench", "--dist", token, "--m", 1000, "--n", 1000, "--p-list", "1,2,4",
                           "--reps", 3, "--seed", 5, "--simulated", "--csv", csv)
        assert code == 0, err
        lines = csv.read_text().splitlines()
        assert lines[0] == "dist,seed,m,n,p,rep,wall_ns,comparisons,max_block,min_block,verified,speedup"
        rows = [r.split(",") for r in lines[1:]]
        assert len(rows) == 9
        assert all(r[10] == "1" for r in rows)
        assert all(r[0] == token and r[1] == "5" for r in rows)
        assert rows[0][-1] == "1"
        expect = golden[f"clibench__{token}__counts"]
        for i, r in enumerate(rows):
            assert int(r[7]) == int(expect[i // 3]), (token, i)


@pytest.mark.gpu
def test_sort_command(tmp_path):
    rng = np.random.default_rng(4)
    keys = [int(x) for x in rng.integers(0, 2**64 - 1, 50_000, dtype=np.uint64)]
    fin = crmg_file(tmp_path / "in.bin", keys)
    out = tmp_path / "sorted.bin"
    code, stdout, _ = run("sort", fin, out)
    assert code == 0 and stdout == "sorted 50000 keys\n"
    assert read_crmg(out) == sorted(keys)
