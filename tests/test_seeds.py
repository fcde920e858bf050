"""Native SeedSequence / PCG64 / permutation streams equal numpy's (host code, no GPU).

The reference draws its jitter streams and surrogate permutations with numpy
(inference.py:41-49, 101-102, 148, 161-172; ksg.py:55); csrc/seeds.cu restates
those algorithms.  These tests pin the restatement bit-for-bit against numpy
for 10k+ seeds, including multi-word (>= 2**32) master seeds and spawned
SeedSequences.
"""

import numpy as np
import pytest

from paper_1401_4068_b200 import seeds
from paper_1401_4068_b200.inference import draw_permutation

MASK = (1 << 64) - 1


def _np_state(seed):
    st = np.random.PCG64(seed).state["state"]
    return (st["state"] >> 64, st["state"] & MASK, st["inc"] >> 64, st["inc"] & MASK)


def test_jitter_states_match_numpy_10k():
    rng = np.random.default_rng(7)
    master = [0, 1, 12345, 2**32 - 1, 2**32, 2**40 + 3, 10**20]
    for m in master:
        us = rng.integers(0, 64, size=1500)
        ids = rng.integers(0, 2**31, size=1500)
        ids[:5] = [0, 1, 2, 2**32 - 1, 0]
        got = seeds.jitter_states(m, us, ids)
        for i in range(0, 1500, 1 if m == 0 else 7):
            want = _np_state(np.random.SeedSequence((m, int(us[i]), int(ids[i]))))
            assert tuple(int(v) for v in got[i]) == want, (m, us[i], ids[i])


def test_jitter_states_wide_columns():
    # column values >= 2**32 take the per-item word-list path
    got = seeds.jitter_states(3, [2**33 + 1, 5], [7, 2**35])
    assert tuple(int(v) for v in got[0]) == _np_state(np.random.SeedSequence((3, 2**33 + 1, 7)))
    assert tuple(int(v) for v in got[1]) == _np_state(np.random.SeedSequence((3, 5, 2**35)))


def test_pcg_states_of_seed_objects():
    parent = np.random.SeedSequence(99)
    cases = [0, 5, 2**64 + 9, (1, 2), [3, 4, 5, 6, 7, 8], np.random.SeedSequence((4, 5)),
             np.random.SeedSequence(), *parent.spawn(3), *np.random.SeedSequence((1, 2)).spawn(2)]
    got = seeds.pcg_states(cases)
    for s, g in zip(cases, got):
        assert tuple(int(v) for v in g) == _np_state(np.random.default_rng(s).bit_generator._seed_seq
                                                     if not isinstance(s, np.random.SeedSequence)
                                                     else s)
    assert seeds.entropy_words(np.random.default_rng(1)) is None
    assert seeds.entropy_words(np.random.SeedSequence(1, pool_size=8)) is None


@pytest.mark.parametrize("reps", [2, 3, 5, 17, 50, 250, 500])
@pytest.mark.parametrize("strict", [True, False])
def test_permutations_match_numpy(reps, strict):
    count = 1500 if reps <= 50 else 300
    for master in (0, 2**36 + 1):
        got = seeds.surrogate_permutations(master, count, reps, strict)
        for i in range(count):
            want = draw_permutation(reps, np.random.SeedSequence((master, i)), strict).permutation
            assert np.array_equal(got[i], want), (reps, strict, master, i)


def test_permutation_errors():
    with pytest.raises(Exception, match="R >= 2"):
        seeds.surrogate_permutations(0, 3, 1, True)
    assert seeds.surrogate_permutations(0, 2, 1, False).tolist() == [[0], [0]]
    assert seeds.surrogate_permutations(0, 0, 5, True).shape == (0, 5)
