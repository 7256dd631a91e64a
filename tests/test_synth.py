"""The seeded input generators (synth/) build bitwise the same matrices with their multi-threaded
torch sorting kernels as with plain numpy (synth._argsort_stable / _unique / _searchsorted_right),
on sizes large enough for the fast path to engage (> 2^20 keys)."""
import hashlib

import numpy as np

import synth


def _digest(p):
    h = hashlib.sha1()
    for a in (p.Q.row_ptr, p.Q.col, p.Q.val, p.b):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_fast_sort_paths_bitwise_numpy(monkeypatch):
    cases = [(3, 0.15), (4, 0.05)]  # ER n = 150k (2.4M edge keys), Chung-Lu n = 200k
    fast = [_digest(synth.config_problem(c, s)) for c, s in cases]
    monkeypatch.setattr(synth, "_FAST", False)
    slow = [_digest(synth.config_problem(c, s)) for c, s in cases]
    assert fast == slow
