"""The fast evaluator's closed-form 1F1B level schedule and the single-slot
channel property that lets a stage read only its neighbours' last channel
value (hp_core.cuh, hp_kernels.cu eval_item_fast), checked against the
counter-driven unit-time ASAP schedule of the reference's op order
(sim.cpp:43-59, 101-104)."""
from __future__ import annotations

import pytest


def asap(P, M, gpipe):
    nf = [0] * P
    nb = [0] * P
    lev = 0
    done = 0
    bad = 0
    F, Bk = {}, {}
    w = [min(P - i, M) for i in range(P)]
    while done < 2 * P * M:
        snf, snb = nf[:], nb[:]
        prog = False
        for i in range(P):
            if gpipe:
                if nf[i] < M:
                    isf = True
                elif nb[i] < M:
                    isf = False
                else:
                    continue
            else:
                if nf[i] < w[i] or (nf[i] < M and nb[i] > nf[i] - w[i]):
                    isf = True
                elif nb[i] < M:
                    isf = False
                else:
                    continue
            if isf:
                if i > 0 and not snf[i - 1] > nf[i]:
                    continue
                if i > 0 and snf[i - 1] != nf[i] + 1:
                    bad += 1
                F[(i, nf[i])] = lev
                nf[i] += 1
            else:
                if i < P - 1 and not snb[i + 1] > nb[i]:
                    continue
                if i < P - 1 and snb[i + 1] != nb[i] + 1:
                    bad += 1
                Bk[(i, nb[i])] = lev
                nb[i] += 1
            done += 1
            prog = True
        assert prog
        lev += 1
    return bad, lev, F, Bk


@pytest.mark.parametrize("gpipe", [False, True])
def test_single_slot_property(gpipe):
    for P in range(1, 19):
        for M in list(range(1, 25)) + [40]:
            bad, _, _, _ = asap(P, M, gpipe)
            assert bad == 0, (P, M)


def test_closed_form_levels():
    for P in range(1, 21):
        for M in range(P, P + 22):
            _, T, F, Bk = asap(P, M, False)
            assert T == 2 * (M + P - 1)
            for (i, m), t in F.items():
                assert t == (i + m if m < P - i else 2 * m + i), (P, M, i, m)
            for (i, j), t in Bk.items():
                assert t == 2 * P - 1 - i + 2 * j, (P, M, i, j)


def test_gpipe_closed_form_levels():
    """GPipe (sim.cpp:46-50): F(i,m) at level i+m, B(i,j) at 2P-2-i+M+j, so
    every forward runs before every backward (levels [0, M+P-2] then
    [M+P-1, 2M+2P-3]) — the two wavefronts of hp_kernels.cu
    eval_item_generic's GPipe path."""
    for P in range(1, 21):
        for M in range(1, 30):
            _, T, F, Bk = asap(P, M, True)
            assert T == 2 * (M + P - 1)
            for (i, m), t in F.items():
                assert t == i + m, (P, M, i, m)
            for (i, j), t in Bk.items():
                assert t == 2 * P - 2 - i + M + j, (P, M, i, j)
            assert max(F.values()) < min(Bk.values())
