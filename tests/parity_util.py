"""Tolerances of the north star (BASELINE.json) and comparison helpers."""

import numpy as np

TWO_PI = 2.0 * np.pi
LAB_ATOL = 1e-4                 # absolute, on L*, a*, b*
NORM_ATOL = 1e-5                # on normalised H/S/I and SCT components
SCT_SCALE = np.array([255.0 * np.sqrt(3.0), np.pi / 2, np.pi / 2])


def nan_mask_equal(a, b):
    np.testing.assert_array_equal(np.isnan(a), np.isnan(b))


def check_lab(got, ref, atol=LAB_ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    assert np.all(err <= atol), f"max |dLab| = {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"
    return float(err.max())


def check_hsi(got, ref, atol=NORM_ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nan_mask_equal(got[..., 0], ref[..., 0])
    d = np.abs(got[..., 0] - ref[..., 0])
    d = np.where(np.isnan(d), 0.0, np.minimum(d, TWO_PI - d)) / TWO_PI   # circular, normalised
    e = np.stack([d, np.abs(got[..., 1] - ref[..., 1]), np.abs(got[..., 2] - ref[..., 2])], -1)
    assert np.all(e <= atol), f"max normalised |dHSI| = {e.max():.3e}"
    return float(e.max())


def check_sct(got, ref, atol=NORM_ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nan_mask_equal(got[..., 2], ref[..., 2])
    e = np.abs(got - ref) / SCT_SCALE
    e = np.where(np.isnan(e), 0.0, e)
    assert np.all(e <= atol), f"max normalised |dSCT| = {e.max():.3e}"
    return float(e.max())


CHECK = {"lab": check_lab, "hsi": check_hsi, "sct": check_sct}


def check_figure(got_avg, got_max, ref_avg, ref_max, avg_rtol=1e-3, max_rtol=1e-2, floor=0.0):
    """mean within 0.1 %, max within 1 %, each with an absolute floor."""
    assert abs(got_avg - ref_avg) <= max(avg_rtol * abs(ref_avg), floor), (got_avg, ref_avg)
    assert abs(got_max - ref_max) <= max(max_rtol * abs(ref_max), floor), (got_max, ref_max)
