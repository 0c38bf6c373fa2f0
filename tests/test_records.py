"""Run records, frame files and post-solve analysis (SURVEY.md §8(f) ranks 1
and 3): ports of the reference's test_io.cpp and the analysis cases of
test_analysis.cpp (paths under /root/reference/proj/tests), plus bit-exact
checks of the GPU magnitudes against the oracle."""
import cmath
import json
import math
import os
import tempfile

import numpy as np
import pytest

from paper_2207_06374_b200 import abi
from paper_2207_06374_b200 import records as rec
from tests import oracle_ffi as orc

C, R = abi.COMPLEX, abi.REAL


def sic_2_4():
    """support.hpp:22-35 (interleaved column-major)."""
    cols = [[1.0, 0.0]]
    c, s = math.sqrt(1.0 / 3.0), math.sqrt(2.0 / 3.0)
    for k in range(3):
        z = cmath.rect(s, 2.0 * 3.14159265358979323846 * k / 3.0)
        cols.append([complex(c, 0.0), z])
    f = []
    for col in cols:
        for v in col:
            v = complex(v)
            f += [v.real, v.imag]
    return np.array(f)


def sic_3_9():
    """support.hpp:39-55."""
    fid = [0.0, 1.0 / math.sqrt(2.0), -1.0 / math.sqrt(2.0)]
    t = 2.0 * 3.14159265358979323846 / 3.0
    f = np.zeros(2 * 3 * 9)
    for a in range(3):
        for b in range(3):
            col = 3 * a + b
            for j in range(3):
                v = cmath.rect(1.0, t * b * j) * fid[(j - a + 3) % 3]
                f[col * 6 + 2 * j] = v.real
                f[col * 6 + 2 * j + 1] = v.imag
    return f


def identity_frame(d):
    f = np.zeros(2 * d * d)
    for j in range(d):
        f[j * 2 * d + 2 * j] = 1.0
    return f


# ------------------------------------------------------------------ CPU: files and bounds
def test_frame_json_round_trips_bit_exactly():  # test_io.cpp:23-29
    f, _ = orc.random_frames(C, 3, 7, 21, 0, 1)
    back, d, N = rec.frame_from_json(json.loads(json.dumps(rec.frame_to_json(f[0], 3, 7))))
    assert (d, N) == (3, 7) and np.array_equal(back.view(np.uint64), f[0].view(np.uint64))


def test_frame_csv_round_trips_bit_exactly():  # test_io.cpp:31-36
    f, _ = orc.random_frames(C, 4, 5, 22, 0, 1)
    back, d, N = rec.frame_from_csv(rec.frame_to_csv(f[0], 4, 5))
    assert (d, N) == (4, 5) and np.array_equal(back.view(np.uint64), f[0].view(np.uint64))


def test_real_frames_are_written_with_zero_imaginary_parts():
    f, _ = orc.random_frames(R, 3, 6, 5, 0, 1)
    back, d, N = rec.frame_from_csv(rec.frame_to_csv(f[0], 3, 6, R))
    assert np.array_equal(back[0::2], f[0]) and not back[1::2].any()


def test_frame_file_save_and_load_by_extension():  # test_io.cpp:38-52
    f, _ = orc.random_frames(C, 2, 6, 23, 0, 1)
    with tempfile.TemporaryDirectory() as tmp:
        for name in ("frame.json", "frame.csv"):
            path = os.path.join(tmp, name)
            rec.save_frame(path, f[0], 2, 6)
            back, d, N = rec.load_frame(path)
            assert (d, N) == (2, 6) and np.array_equal(back, f[0])


def test_malformed_frame_files_raise():  # test_io.cpp:54-62
    with pytest.raises(rec.FileFormatError):
        rec.frame_from_json({"d": 2})
    with pytest.raises(rec.FileFormatError):
        rec.frame_from_json({"d": 2, "N": 1, "columns": [[1.0, 0.0]]})  # column too short
    with pytest.raises(rec.FileFormatError):
        rec.frame_from_csv("1.0,2.0\n")  # odd rows
    with pytest.raises(rec.FileFormatError):
        rec.frame_from_csv("1.0,x\n0.0,0.0\n")
    with pytest.raises(rec.FileFormatError):
        rec.load_frame("/nonexistent/path/frame.json")


def test_full_precision_text_round_trip():  # test_io.cpp:110-116
    for v in (0.1, 1.0 / 3.0, 0.5773502691896258, 1e-300, -0.7071067811865476):
        assert float(rec.full_precision(v)) == v


def test_bounds_report_closed_forms():  # test_analysis.cpp:36-54, 56-63
    b39 = rec.bounds_report(3, 9)
    assert abs(b39["welch"] - 0.5) <= 1e-15 and b39["orthoplex"] is None and b39["levenshtein"] is None
    assert b39["gerzon_max"] == 9 and b39["best_applicable"] == b39["welch"]
    b25 = rec.bounds_report(2, 5)
    assert abs(b25["orthoplex"] - 1.0 / math.sqrt(2.0)) <= 1e-12
    assert abs(b25["levenshtein"] - 2.0 / 3.0) <= 1e-12
    assert b25["best_applicable"] == max(b25["welch"], b25["orthoplex"], b25["levenshtein"])
    for d in range(2, 9):
        assert abs(rec.bounds_report(d, d + 1)["welch"] - 1.0 / d) <= 1e-15
    assert rec.bounds_report(4, 4)["welch"] == 0.0
    with pytest.raises(ValueError):
        rec.bounds_report(4, 3)
    # config 2: Levenshtein binds
    assert abs(rec.bounds_report(2, 100)["best_applicable"] - 0.812320100) < 1e-9


def test_cluster_sorted_is_the_reference_single_linkage():  # frame.hpp:96-118
    v = np.array([0.1, 0.10005, 0.1001, 0.5, 0.50002, 0.9])
    means = rec.cluster_sorted(v, 1e-4)
    ref, s, k, last = [], 0.0, 0, 0.0
    for x in v:  # the reference's loop, sequential sums
        if k > 0 and x - last > 1e-4:
            ref.append(s / k)
            s, k = 0.0, 0
        s += x
        last = x
        k += 1
    ref.append(s / k)
    assert np.array_equal(means, np.array(ref))
    with pytest.raises(ValueError):
        rec.cluster_sorted(v, 0.0)


# ------------------------------------------------------------------ GPU: analysis kernels
@pytest.mark.gpu
@pytest.mark.parametrize("field,d,N", [(C, 2, 4), (C, 3, 9), (C, 2, 100), (R, 4, 10), (C, 128, 300)])
def test_magnitudes_bit_exact_vs_oracle(field, d, N):
    f = orc.random_test_frame(field, d, N, 77)
    m = rec.offdiagonal_magnitudes(f, d, N, field)
    mo = orc.offdiag_magnitudes(field, d, N, f)
    assert np.array_equal(m.view(np.uint64), mo.view(np.uint64))
    s = rec.offdiagonal_magnitudes(f, d, N, field, sort=True)
    assert np.array_equal(s, np.sort(mo))
    mu, arg, _ = orc.coherence(field, d, N, f)
    assert m.max() == mu and int(np.argmax(m)) == arg


@pytest.mark.gpu
def test_magnitudes_normalize_and_zero_column():
    f = orc.random_test_frame(C, 3, 8, 5) * 2.5
    m = rec.offdiagonal_magnitudes(f, 3, 8, C, normalize=True)
    assert m.max() <= 1.0 + 1e-15
    f[2 * 6:3 * 6] = 0.0
    from paper_2207_06374_b200.api import ZeroColumnError
    with pytest.raises(ZeroColumnError):
        rec.offdiagonal_magnitudes(f, 3, 8, C, normalize=True)


@pytest.mark.gpu
def test_analytic_equiangular_fixtures():  # test_analysis.cpp:24-34
    s24 = rec.gram_summary(sic_2_4(), 2, 4, C, 1e-9)
    assert s24["angle_spectrum"].size == 1 and abs(s24["angle_spectrum"][0] - 1.0 / math.sqrt(3.0)) <= 1e-12
    s39 = rec.gram_summary(sic_3_9(), 3, 9, C, 1e-9)
    assert s39["offdiag_mags"].size == 36
    assert s39["angle_spectrum"].size == 1 and abs(s39["angle_spectrum"][0] - 0.5) <= 1e-12


@pytest.mark.gpu
def test_tightness_check():  # test_analysis.cpp:71-86
    ok, dev = rec.check_tight(identity_frame(3), 3, 3, C, 1e-12)
    assert ok and dev == 0.0
    ok, dev = rec.check_tight(sic_2_4(), 2, 4, C, 1e-10)
    assert ok and dev <= 1e-10
    rep = np.zeros(2 * 2 * 3)
    rep[0::4] = 1.0  # three copies of e_0
    ok, dev = rec.check_tight(rep, 2, 3, C, 1e-6)
    assert not ok and abs(dev - 1.5) <= 1e-12


@pytest.mark.gpu
def test_etf_certificates():  # test_analysis.cpp:88-105
    assert rec.check_etf(sic_2_4(), 2, 4, C, 1e-6)["kind"] == "etf"
    assert rec.check_etf(identity_frame(4), 4, 4, C, 1e-10)["kind"] == "etf"
    f, _ = orc.random_frames(C, 3, 5, 0, 0, 1)
    assert rec.check_etf(f[0], 3, 5, C, 1e-4)["kind"] == "none"
    for frame, d, N in ((sic_2_4(), 2, 4), (sic_3_9(), 3, 9)):
        assert rec.check_etf(frame, d, N, C, 1e-6)["kind"] == "etf"
        mu = orc.coherence(C, d, N, frame)[0]
        assert abs(mu - rec.bounds_report(d, N)["welch"]) <= 2e-6


@pytest.mark.gpu
def test_certificates_of_the_sic():
    kinds = {c["kind"] for c in rec.certificates(sic_2_4(), 2, 4, C, 1e-6)}
    assert {"tight_frame", "etf", "one_distance", "welch_equality"} <= kinds


@pytest.mark.gpu
def test_run_records_round_trip_and_stay_self_consistent():  # test_io.cpp:64-89
    cfg = abi.default_cfg(C, 2, 4, 200, eps_target=1e-6)
    res = rec.solve(cfg, restarts=3, seed=4711)
    record = rec.make_run_record("trstmi", res, rec.solver_config_to_json(cfg, 3, 4711),
                                 rec.iso8601_utc_now(), rec.iso8601_utc_now())
    reparsed = json.loads(json.dumps(record))
    assert reparsed == record
    assert json.dumps(json.loads(json.dumps(reparsed))) == json.dumps(reparsed)
    frame, d, N = rec.frame_from_json(record["best_frame"])
    assert abs(orc.coherence(C, d, N, frame, normalize=True)[0] - record["best_coherence"]) <= 1e-12
    assert record["schema_version"] == 1 and record["method"] == "trstmi"
    assert len(record["per_restart"]) == 3
    assert abs(record["bounds"]["welch"] - rec.bounds_report(2, 4)["welch"]) <= 1e-15
    # the (2,4) optimum is the SIC: mu = 1/sqrt(3) (README.md:139-146)
    assert abs(record["best_coherence"] - 1.0 / math.sqrt(3.0)) < 1e-6
    assert [r["seed"] for r in record["per_restart"]] == [orc.mix_seed(4711, i) for i in range(3)]


@pytest.mark.gpu
def test_identical_solves_give_identical_records_modulo_timing():  # test_io.cpp:91-108
    cfg = abi.default_cfg(C, 2, 3, 200, eps_target=1e-5)

    def without_timing():
        r = rec.solve(cfg, restarts=2, seed=31)
        j = rec.make_run_record("trstmi", r, rec.solver_config_to_json(cfg, 2, 31), "T0", "T1")
        del j["timestamps"], j["wall_time_seconds"]
        return j

    assert without_timing() == without_timing()


# ------------------------------------------------------------------ GPU: MISO codebook distortion
@pytest.mark.gpu
@pytest.mark.parametrize("d,N,samples,seed", [(2, 4, 50000, 99), (3, 9, 20000, 7), (2, 1, 9000, 5), (4, 40, 5000, 3)])
def test_distortion_matches_the_oracle(d, N, samples, seed):
    book = sic_2_4() if (d, N) == (2, 4) else (sic_3_9() if (d, N) == (3, 9) else
                                                  orc.random_frames(C, d, N, 11, 0, 1)[0][0])
    if (d, N) == (2, 1):
        book = np.array([1.0, 0.0, 0.0, 0.0])
    g = rec.distortion_mc(book, d, N, samples, seed)
    eo, so = orc.distortion_mc(d, N, book, samples, seed)
    # the integer SplitMix64 streams are identical; CUDA and glibc log/sin/cos
    # differ by an ulp or two, so the estimates agree to rounding
    assert abs(g["estimate"] - eo) <= 1e-12 * max(1.0, abs(eo))
    assert abs(g["std_error"] - so) <= 1e-9 * max(so, 1e-300)


@pytest.mark.gpu
def test_distortion_of_a_single_codeword_in_d2_is_one_half():  # test_beamforming.cpp:107-126
    est = rec.distortion_mc(np.array([1.0, 0.0, 0.0, 0.0]), 2, 1, 200000, 5)
    assert abs(est["estimate"] - 0.5) <= 4.0 * est["std_error"]


@pytest.mark.gpu
def test_distortion_estimates_are_deterministic():  # test_beamforming.cpp:128-137
    a = rec.distortion_mc(sic_2_4(), 2, 4, 50000, 99)
    b = rec.distortion_mc(sic_2_4(), 2, 4, 50000, 99)
    assert a == b


@pytest.mark.gpu
def test_standard_error_scales_like_inverse_sqrt_samples():  # test_beamforming.cpp:139-147
    small = rec.distortion_mc(sic_2_4(), 2, 4, 40000, 3)
    large = rec.distortion_mc(sic_2_4(), 2, 4, 160000, 3)
    assert 0.0 <= small["estimate"] <= 1.0
    assert abs(small["std_error"] / large["std_error"] - 2.0) <= 0.6


@pytest.mark.gpu
def test_codebook_orderings():  # test_beamforming.cpp:149-180
    big = orc.random_frames(C, 2, 12, 246, 0, 1)[0][0]
    small = big[:5 * 4]
    ds, db = rec.distortion_mc(small, 2, 5, 100000, 31), rec.distortion_mc(big, 2, 12, 100000, 31)
    assert db["estimate"] <= ds["estimate"] + 2.0 * (ds["std_error"] + db["std_error"])
    basis, sic = rec.distortion_mc(identity_frame(2), 2, 2, 200000, 13), rec.distortion_mc(sic_2_4(), 2, 4, 200000, 13)
    assert sic["estimate"] + 3.0 * (sic["std_error"] + basis["std_error"]) < basis["estimate"]
    dense = orc.random_frames(C, 2, 1000, 135, 0, 1)[0][0]
    sparse = orc.random_frames(C, 2, 10, 135, 0, 1)[0][0]
    dd, dsp = rec.distortion_mc(dense, 2, 1000, 20000, 77), rec.distortion_mc(sparse, 2, 10, 20000, 77)
    assert dd["estimate"] < dsp["estimate"] and dd["estimate"] < 0.01
