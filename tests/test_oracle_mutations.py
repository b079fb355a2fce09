"""Mutation check of the oracle's pins (VERDICT r1 "done when"): each plausible slip in
oracle.c — a transposed R(q), a flipped sign in the EWA Jacobian's third column, a wrong
factor in its derivative, a sign error in the SH basis used for the clamp decision — is
compiled into a separate copy of the oracle, and at least one pin of tests/test_oracle.py
must fail against it.  The fp32 decision chain and the fp64 value chain are written
separately (oracle.c header), so each is mutated on its own."""
import math
import os

import numpy as np
import pytest

import oracle
import test_oracle as T

SRC = open(os.path.join(os.path.dirname(oracle.__file__), "oracle.c")).read()

MUTATIONS = {
    "activate32: R transposed": [
        ("R[0][1] = 2.0f * fmaf(x, y, -(w * z));", "R[0][1] = 2.0f * fmaf(x, y, w * z);"),
        ("R[0][2] = 2.0f * fmaf(x, z, w * y);", "R[0][2] = 2.0f * fmaf(x, z, -(w * y));"),
        ("R[1][0] = 2.0f * fmaf(x, y, w * z);", "R[1][0] = 2.0f * fmaf(x, y, -(w * z));"),
        ("R[1][2] = 2.0f * fmaf(y, z, -(w * x));", "R[1][2] = 2.0f * fmaf(y, z, w * x);"),
        ("R[2][0] = 2.0f * fmaf(x, z, -(w * y));", "R[2][0] = 2.0f * fmaf(x, z, w * y);"),
        ("R[2][1] = 2.0f * fmaf(y, z, w * x);", "R[2][1] = 2.0f * fmaf(y, z, -(w * x));"),
    ],
    "activate64: R transposed": [
        ("R[0][1] = 2 * (x * y - w * z); R[0][2] = 2 * (x * z + w * y);",
         "R[0][1] = 2 * (x * y + w * z); R[0][2] = 2 * (x * z - w * y);"),
        ("R[1][0] = 2 * (x * y + w * z);", "R[1][0] = 2 * (x * y - w * z);"),
        ("R[1][2] = 2 * (y * z - w * x);", "R[1][2] = 2 * (y * z + w * x);"),
        ("R[2][0] = 2 * (x * z - w * y); R[2][1] = 2 * (y * z + w * x);",
         "R[2][0] = 2 * (x * z + w * y); R[2][1] = 2 * (y * z - w * x);"),
    ],
    "project32: J02 sign": [("J02 = -(c->fx * uxc) / tz;", "J02 = (c->fx * uxc) / tz;")],
    "project32: J12 sign": [("J12 = -(c->fy * uyc) / tz;", "J12 = (c->fy * uyc) / tz;")],
    "project64: J02 sign": [("p->J[0][2] = -fx * uxc / tz;", "p->J[0][2] = fx * uxc / tz;")],
    "project64: J12 sign": [("p->J[1][2] = -fy * uyc / tz;", "p->J[1][2] = fy * uyc / tz;")],
    "project32: R_v row swapped in T": [("T1[j] = fmaf(J12, R[6 + j], J11 * R[3 + j]);",
                                         "T1[j] = fmaf(J12, R[6 + j], J11 * R[j]);")],
    "gauss_backward: dJ02/dtz factor 2 -> 1": [("dt[2] += 2 * fx * tx / (tz2 * tz) * dJ[0][2];",
                                                "dt[2] += fx * tx / (tz2 * tz) * dJ[0][2];")],
    "color32: Y1 sign": [("Y[1] = -0.4886025119029199f * y;", "Y[1] = 0.4886025119029199f * y;")],
    "color32: Y12 order": [("Y[12] = (0.3731763325901154f * z) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);",
                            "Y[12] = (0.3731763325901154f * z) * ((2.0f * xx - 3.0f * zz) - 3.0f * yy);")],
}

PINS = [
    T.test_P1_axis_swap_through_projection,
    lambda: [T.test_P1b_rotation_matches_rodrigues_through_three_cameras(a, t) for a, t in T.ROT_CASES],
    T.test_P2b_offaxis_ewa_matches_pinhole_linearisation,
    T.test_P2c_offaxis_ewa_monte_carlo,
    T.test_P3_isotropic_on_axis_conic_and_radius,
    T.test_P17b_sh_clamp_decision_is_the_sign_of_the_colour,
    lambda: T.test_P10_all_gradients_match_finite_differences(1),
]


@pytest.mark.parametrize("name", list(MUTATIONS))
def test_a_pin_fails_on_the_mutated_oracle(name, tmp_path):
    src = SRC
    for old, new in MUTATIONS[name]:
        assert src.count(old) == 1, f"mutation site not unique: {old}"
        src = src.replace(old, new)
    lib = oracle.build_variant(src, str(tmp_path / "libmut.so"))
    failed = []
    try:
        oracle.use_library(lib)
        for pin in PINS:
            try:
                pin()
            except AssertionError:
                failed.append(getattr(pin, "__name__", "pin"))
    finally:
        oracle.use_library(None)
    assert failed, f"no pin detects '{name}'"


def test_unmutated_oracle_passes_the_same_pins(tmp_path):
    lib = oracle.build_variant(SRC, str(tmp_path / "libsame.so"))
    try:
        oracle.use_library(lib)
        for pin in PINS:
            pin()
    finally:
        oracle.use_library(None)
