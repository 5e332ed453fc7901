"""Pins for the parity metric itself, ``oracle.rowwise_rel_err`` [reading c12].

Every bf16 / fp32 parity assertion in this repo goes through

    err(z, zref) = max_m ||z_m - zref_m||_inf / max(||zref_m||_inf, 1e-30)

(SPEC.md:432 uses the inf-norm relative error of a vector; the row-wise form is
reading c12 in DESIGN.md: one token's output is one vector, PAPER.md:14 defines the
norm per vector).  The values below are computed by hand (exact binary fractions where
possible), so a plausible mistake in the metric -- a global instead of a per-row
denominator, normalising by the kernel's row instead of the oracle's, a mean instead
of a max over rows, an L1/L2 norm instead of the inf-norm, a dropped ``abs`` or a
missing floor -- changes at least one of them.  The mutants at the end are those
mistakes written out; each must disagree with a hand value.
"""
import math

import numpy as np
import pytest

from oracle import flashnorm_oracle as O

TOL_BF16 = 2e-2   # BASELINE.json north_star: bf16-in / fp32-accumulate


# (z, zref, hand value, what it pins)
HAND_CASES = [
    # one row, exact binary fractions: |5 - 4| / |4| = 1/4 (normalised by zref, not z: 1/5)
    ([[5.0, 0.0]], [[4.0, 0.0]], 0.25, "orientation: denominator is the reference row"),
    # inf-norm inside the row: diff (0.25, 0.25), ||zref||_inf = 4 -> 1/16
    #   (L1 would give 0.5 / 5 = 0.1, L2 sqrt(0.125)/sqrt(17) = 0.0857...)
    ([[1.25, 4.25]], [[1.0, 4.0]], 0.0625, "inf-norm over the row"),
    # dropped abs: z below zref -> |0 - 1| / 1 = 1 (max(z - zref) would give 0)
    ([[0.0, 0.0]], [[1.0, 0.0]], 1.0, "absolute difference"),
    # two rows of very different magnitude; only the small row is wrong:
    #   row 0: 0 / 2 = 0;  row 1: |1.5e-3 - 1e-3| / 1e-3 = 0.5  -> 0.5
    #   (a global inf-norm denominator gives 5e-4 / 2 = 2.5e-4)
    ([[2.0, 1.0], [1.5e-3, 0.0]], [[2.0, 1.0], [1e-3, 0.0]], 0.5, "per-row denominator"),
    # max over rows, not mean: row errors 1/2 and 0 -> 1/2 (mean 1/4)
    ([[3.0, 0.0], [8.0, 8.0]], [[2.0, 0.0], [8.0, 8.0]], 0.5, "max over rows"),
    # the floor: an all-zero reference row and an all-zero result row -> 0 (no 0/0 NaN)
    ([[0.0, 0.0], [1.0, 1.0]], [[0.0, 0.0], [1.0, 1.0]], 0.0, "floor, 0/0"),
    # the floor: reference row zero, result row not -> 1e-3 / 1e-30 = 1e27 (caught, not hidden)
    ([[1e-3, 0.0]], [[0.0, 0.0]], 1e27, "floor value 1e-30"),
]


@pytest.mark.parametrize("z,zref,want,what", HAND_CASES, ids=[c[3] for c in HAND_CASES])
def test_rowwise_rel_err_hand_values(z, zref, want, what):
    got = O.rowwise_rel_err(np.array(z), np.array(zref))
    assert math.isclose(got, want, rel_tol=1e-12), (what, got, want)


def test_rowwise_rel_err_empty_and_shapes():
    assert O.rowwise_rel_err(np.zeros((0, 4)), np.zeros((0, 4))) == 0.0
    # a single vector is one row
    assert math.isclose(O.rowwise_rel_err(np.array([3.0, 4.5]), np.array([3.0, 4.0])), 0.125)
    # bf16-looking inputs are widened to fp64 before subtracting (no fp32 cancellation)
    z = np.array([[1.0 + 2.0 ** -30]], dtype=np.float64)
    assert math.isclose(O.rowwise_rel_err(z, np.array([[1.0]])), 2.0 ** -30, rel_tol=1e-9)


def test_rowwise_rel_err_nan_is_not_hidden():
    """A NaN in the result must not read as a pass (np.max propagates NaN; NaN <= tol is False)."""
    got = O.rowwise_rel_err(np.array([[np.nan, 1.0]]), np.array([[1.0, 1.0]]))
    assert not (got <= TOL_BF16)


def test_low_energy_row_fault_fails_at_bf16_tolerance():
    """A kernel wrong ONLY on a low-energy row (5 % off on a row 1e-3 the size of the others)
    must fail the 2e-2 bar; under a global denominator it would pass (5e-5 absolute)."""
    rng = np.random.default_rng(7)
    zref = rng.standard_normal((8, 64))
    zref[5] *= 1e-3                      # a low-energy token (the 'lowenergy' input mode)
    z = zref.copy()
    z[5] *= 1.05
    assert O.rowwise_rel_err(z, zref) > TOL_BF16
    assert math.isclose(O.rowwise_rel_err(z, zref), 0.05, rel_tol=1e-9)
    assert _global_denominator(z, zref) < TOL_BF16       # the mutant would hide it


# --- the plausible mistakes, written out; each disagrees with some hand value ------------------

def _global_denominator(z, zref):
    z, zref = np.asarray(z, float), np.asarray(zref, float)
    return float(np.max(np.abs(z - zref)) / max(np.max(np.abs(zref)), 1e-30))


def _kernel_denominator(z, zref):
    return O.rowwise_rel_err(zref, z)


def _mean_over_rows(z, zref):
    z, zref = np.atleast_2d(np.asarray(z, float)), np.atleast_2d(np.asarray(zref, float))
    num = np.max(np.abs(z - zref), axis=-1)
    return float(np.mean(num / np.maximum(np.max(np.abs(zref), axis=-1), 1e-30)))


def _l1_row(z, zref):
    z, zref = np.atleast_2d(np.asarray(z, float)), np.atleast_2d(np.asarray(zref, float))
    num = np.sum(np.abs(z - zref), axis=-1)
    return float(np.max(num / np.maximum(np.sum(np.abs(zref), axis=-1), 1e-30)))


def _no_abs(z, zref):
    z, zref = np.atleast_2d(np.asarray(z, float)), np.atleast_2d(np.asarray(zref, float))
    num = np.max(z - zref, axis=-1)
    return float(np.max(num / np.maximum(np.max(np.abs(zref), axis=-1), 1e-30)))


def _no_floor(z, zref):
    z, zref = np.atleast_2d(np.asarray(z, float)), np.atleast_2d(np.asarray(zref, float))
    with np.errstate(invalid="ignore", divide="ignore"):
        return float(np.max(np.max(np.abs(z - zref), axis=-1) / np.max(np.abs(zref), axis=-1)))


@pytest.mark.parametrize("mutant", [_global_denominator, _kernel_denominator, _mean_over_rows,
                                    _l1_row, _no_abs, _no_floor])
def test_each_mutant_misses_a_hand_value(mutant):
    misses = 0
    for z, zref, want, _ in HAND_CASES:
        got = mutant(np.array(z), np.array(zref))
        if not (math.isclose(got, want, rel_tol=1e-12)):
            misses += 1
    assert misses >= 1, mutant.__name__
