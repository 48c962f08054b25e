"""The integer-ulp closed form of K4's chunk-base recurrence (chunk_jump_bits
in csrc/vx_render.cu), restated in numpy and checked against the sequential
FP32 recurrence it replaces: base <- fl(base + adv), render.py:331 (SURVEY.md
Appendix A).  CPU only: the frame parity tests check the kernel itself.
"""
import numpy as np
import pytest

F32 = np.float32


def seq(base, adv, n):
    b = F32(base)
    for _ in range(n):
        b = F32(b + F32(adv))
    return b


def jump_bits(base, adv, J):
    """Line-for-line restatement of chunk_jump_bits (returns base, steps)."""
    ab = int(np.array(adv, F32).view(np.uint32))
    ea = ab >> 23
    ma = (ab & 0x7FFFFF) | 0x800000
    b = int(np.array(base, F32).view(np.uint32))
    done = 0
    while done < J:
        eb = b >> 23
        sh = eb - ea
        if sh < 1 or sh > 23 or eb > 253 or ea < 1:
            break
        half = 1 << (sh - 1)
        if (ma & (2 * half - 1)) == half:
            break
        A = (ma + half) >> sh
        room = 0x800000 - (b & 0x7FFFFF)
        n = J - done
        if n * A > room:
            n = room // A
        if n == 0:
            b = int(np.array(F32(np.array(b, np.uint32).view(F32) + F32(adv)), F32).view(np.uint32))
            done += 1
        else:
            b += n * A
            done += n
    return np.array(b, np.uint32).view(F32)[()], done


def finish(base, adv, J):
    b, done = jump_bits(base, adv, J)
    return seq(b, adv, J - done), done


@pytest.mark.parametrize("seed", range(4))
def test_jump_equals_sequential_random(seed):
    rng = np.random.default_rng(seed)
    for _ in range(400):
        base = F32(rng.uniform(0.0, 4096.0) * (2.0 ** rng.integers(-6, 3)))
        adv = F32(rng.choice([0.5, 1.0, 2.0, 4.0, 8.0]) * rng.uniform(0.05, 1.5))
        J = int(rng.integers(1, 300))
        got, _ = finish(base, adv, J)
        assert got == seq(base, adv, J), (base, adv, J)


def test_binade_crossings_and_exact_power():
    # sums landing exactly on 2^(e+1) and runs across several binades
    for base in (F32(1023.75), F32(2047.5), F32(255.9375), F32(1.0), F32(3.999)):
        for adv in (F32(0.25), F32(0.1), F32(0.3333333), F32(7.0)):
            for J in (1, 2, 3, 17, 1000):
                got, _ = finish(base, adv, J)
                assert got == seq(base, adv, J), (base, adv, J)


def test_ties_fall_back():
    # adv / ulp(base) = x.5 exactly: the jump refuses, the sequence finishes
    base = F32(1024.0)  # ulp 2^-13
    adv = F32(3 * 2.0 ** -14)  # 1.5 ulp: a tie
    b, done = jump_bits(base, adv, 10)
    assert done == 0 and b == base
    got, _ = finish(base, adv, 10)
    assert got == seq(base, adv, 10)


def test_degenerate_steps_fall_back():
    # adv below half an ulp (base + adv == base) and zero/negative bases
    assert jump_bits(F32(2.0 ** 30), F32(1.0), 5)[1] == 0
    assert jump_bits(F32(0.0), F32(0.5), 5)[1] == 0
    assert jump_bits(F32(-3.0), F32(0.5), 5)[1] == 0
