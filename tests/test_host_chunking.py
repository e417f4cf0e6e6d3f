"""The host pipeline's chunk arithmetic (comerge_cuda.cu, merge_host_pipeline)
restated and checked on the CPU against the oracle: output chunks cut on a
G-element grid, each input window copied from its G-aligned start, and the
chunk merged as the output range [(j0 - sa) + (k0 - sb), +(i1 - i0)) of the
merge of A[sa, j1) and B[sb, k1).  The claim the device path relies on: the
leading elements A[sa, j0) and B[sb, k0) precede every chunk element in the
stable order, so that range is exactly out[i0, i1) -- ties included (the
chunk boundaries fall inside runs of equal keys)."""
import numpy as np
import pytest

G = 64  # elements (256 bytes of 32-bit data), as the device path


def chunks(total, parts):
    chunk = -(-max(-(-total // parts), 1 << 12) // G) * G  # small minimum for the test
    return [min(total, c * chunk) for c in range(-(-total // chunk) + 1)]


@pytest.mark.parametrize("alphabet", [2, 16, 1 << 20])
@pytest.mark.parametrize("shape", [(70_001, 50_003), (5, 90_000), (90_000, 0), (33_333, 33_333)])
def test_chunk_windows_are_exact_output_ranges(port, alphabet, shape):
    rng = np.random.default_rng(alphabet + shape[0])
    m, n = shape
    a = np.sort(rng.integers(0, alphabet, m)).astype(np.int32)
    b = np.sort(rng.integers(0, alphabet, n)).astype(np.int32)
    av = np.arange(m, dtype=np.uint32)
    bv = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
    ek, ev = port.merge(a, b, av, bv)
    cuts = chunks(m + n, 8)
    js = [port.co_rank(i, a, b)[0] for i in cuts]
    for c in range(len(cuts) - 1):
        i0, i1, j0, j1 = cuts[c], cuts[c + 1], js[c], js[c + 1]
        assert i0 % G == 0
        k0, k1 = i0 - j0, i1 - j1
        sa, sb = j0 // G * G, k0 // G * G
        wk, wv = port.merge(a[sa:j1], b[sb:k1], av[sa:j1], bv[sb:k1])
        r0 = (j0 - sa) + (k0 - sb)
        assert np.array_equal(wk[r0:r0 + (i1 - i0)], ek[i0:i1]), c
        assert np.array_equal(wv[r0:r0 + (i1 - i0)], ev[i0:i1]), c
        # the device-to-host copies: the A window's share, rounded to the grid
        h = min(i1, i0 + (j1 - j0 + G // 2) // G * G) - i0
        assert 0 <= h <= i1 - i0 and (i0 + h == i1 or (i0 + h) % G == 0)
