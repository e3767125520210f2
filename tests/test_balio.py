"""Problem-file reader/writer (balio.py:1-97) through libbamg_b200's native parser:
bit-exact round trips, the reference's error classes / messages / line numbers
(restating pkg/tests/test_balio.py), and byte parity of the writer with the
reference's f"{v:.17g}" formatting. Host-only: no GPU needed, except the
BundleProblem round trip marked gpu."""

import numpy as np
import pytest

from paper_2007_01941_b200 import scenes
from paper_2007_01941_b200.balio import BalFormatError, read_bal_arrays, write_bal_arrays


def hand_lines():
    lines = ["2 2 4"]
    lines += ["0 0 1.5 -2.5", "0 1 3.25 4.5", "1 0 -5.5 6.0", "1 1 7.0 -8.0"]
    lines += [f"{0.001 * k}" for k in range(1, 10)]
    lines += [f"{0.002 * k}" for k in range(1, 10)]
    lines += [f"{1.0 + 0.1 * k}" for k in range(6)]
    return lines


def write_lines(path, lines, end="\n"):
    path.write_text(end.join(lines) + end)
    return str(path)


def reference_text(cams, pts, ci, pi, pix):
    """The reference writer's output (balio.py:25-35), restated with Python formatting."""
    out = [f"{cams.shape[0]} {pts.shape[0]} {len(ci)}\n"]
    for c, p, (x, y) in zip(ci, pi, pix):
        out.append(f"{c} {p} {x:.17g} {y:.17g}\n")
    out += [f"{v:.17g}\n" for v in cams.ravel()]
    out += [f"{v:.17g}\n" for v in pts.ravel()]
    return "".join(out)


def test_header_counts_parsed(tmp_path):
    cams, pts, ci, pi, pix = read_bal_arrays(write_lines(tmp_path / "p.txt", hand_lines()))
    assert cams.shape == (2, 9) and pts.shape == (2, 3) and len(ci) == 4
    np.testing.assert_array_equal(ci, [0, 0, 1, 1])
    np.testing.assert_array_equal(pi, [0, 1, 0, 1])
    np.testing.assert_array_equal(pix[0], [1.5, -2.5])
    assert cams[1, 0] == 0.002
    assert pts[1, 2] == 1.5


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_round_trip_is_bit_exact_and_matches_reference_bytes(tmp_path, threads):
    sc = scenes.random_problem(21, n_cameras=4, n_points=12, pixel_noise=0.7)
    arrs = sc.arrays()
    path = tmp_path / "rt.txt"
    write_bal_arrays(path, *arrs, n_threads=threads)
    assert path.read_text() == reference_text(*[np.asarray(a) for a in arrs])
    back = read_bal_arrays(path, n_threads=threads)
    for a, b in zip(arrs, back):
        assert np.array_equal(np.asarray(a), b)
    path2 = tmp_path / "rt2.txt"
    write_bal_arrays(path2, *back)
    assert path.read_bytes() == path2.read_bytes()


def test_round_trip_special_values(tmp_path):
    sc = scenes.random_problem(22, n_cameras=3, n_points=9)
    cams, pts, ci, pi, pix = [np.array(a, copy=True) for a in sc.arrays()]
    cams[0, 0] = -0.0
    cams[1, 8] = 5e-324
    pts[0, 1] = -1e-310
    pix[0, 0] = 1e300
    pix[1, 1] = 1e16
    path = tmp_path / "z.txt"
    write_bal_arrays(path, cams, pts, ci, pi, pix)
    assert path.read_text() == reference_text(cams, pts, ci, pi, pix)
    c2, p2, _, _, x2 = read_bal_arrays(path)
    assert np.signbit(c2[0, 0])
    assert c2[1, 8] == 5e-324
    assert p2[0, 1] == -1e-310
    assert x2[0, 0] == 1e300 and x2[1, 1] == 1e16


def test_many_threads_large_file(tmp_path):
    """Chunk boundaries everywhere: a ~3 MB file parsed with 1 and 8 threads."""
    rng = np.random.default_rng(0)
    nc, npt, k = 50, 20000, 60000
    cams, pts = rng.normal(size=(nc, 9)), rng.normal(size=(npt, 3)) * 1e3
    ci, pi = rng.integers(0, nc, k), rng.integers(0, npt, k)
    pix = rng.normal(size=(k, 2)) * 500
    path = tmp_path / "big.txt"
    write_bal_arrays(path, cams, pts, ci, pi, pix, n_threads=8)
    for t in (1, 8):
        back = read_bal_arrays(path, n_threads=t)
        for a, b in zip((cams, pts, ci, pi, pix), back):
            assert np.array_equal(a, b)


def test_blank_lines_and_crlf(tmp_path):
    lines = hand_lines()
    lines.insert(1, "")
    lines.insert(8, "   ")
    _, _, ci, _, _ = read_bal_arrays(write_lines(tmp_path / "p.txt", lines))
    assert len(ci) == 4
    cams, *_ = read_bal_arrays(write_lines(tmp_path / "q.txt", hand_lines(), end="\r\n"))
    assert cams[1, 0] == 0.002


@pytest.mark.parametrize("n,section", [(1, "observation 0"), (3, "observation 2"), (5, "camera parameters"),
                                       (23, "point coordinates")])
def test_truncated_file_names_missing_section(tmp_path, n, section):
    path = write_lines(tmp_path / "t.txt", hand_lines()[:n])
    with pytest.raises(BalFormatError, match=f"file ends before {section}") as err:
        read_bal_arrays(path)
    assert err.value.lineno == n + 1


def test_header_errors_carry_line_number(tmp_path):
    with pytest.raises(BalFormatError, match="header needs 3 counts, got 2") as err:
        read_bal_arrays(write_lines(tmp_path / "a.txt", ["2 2"]))
    assert err.value.lineno == 1
    with pytest.raises(BalFormatError, match=r"malformed header count in '2 x 4'"):
        read_bal_arrays(write_lines(tmp_path / "b.txt", ["2 x 4"]))
    with pytest.raises(BalFormatError, match="nonnegative"):
        read_bal_arrays(write_lines(tmp_path / "c.txt", ["2 -1 4"]))
    with pytest.raises(BalFormatError, match="file ends before header") as err:
        read_bal_arrays(write_lines(tmp_path / "d.txt", ["", "  "]))
    assert err.value.lineno == 3


def test_observation_errors_carry_line_number(tmp_path):
    lines = hand_lines()
    lines[2] = "0 1 3.25"
    with pytest.raises(BalFormatError, match="observation needs 4 fields, got 3") as err:
        read_bal_arrays(write_lines(tmp_path / "a.txt", lines))
    assert err.value.lineno == 3
    lines = hand_lines()
    lines[3] = "1 0 -5.5 bad"
    with pytest.raises(BalFormatError, match=r"malformed observation '1 0 -5.5 bad'") as err:
        read_bal_arrays(write_lines(tmp_path / "b.txt", lines))
    assert err.value.lineno == 4


def test_index_range_errors(tmp_path):
    lines = hand_lines()
    lines[1] = "2 0 1.5 -2.5"
    with pytest.raises(BalFormatError, match=r"camera index 2 out of range \[0, 2\)"):
        read_bal_arrays(write_lines(tmp_path / "a.txt", lines))
    lines = hand_lines()
    lines[4] = "1 5 7.0 -8.0"
    with pytest.raises(BalFormatError, match=r"point index 5 out of range \[0, 2\)"):
        read_bal_arrays(write_lines(tmp_path / "b.txt", lines))


def test_malformed_scalar_carries_section_and_line(tmp_path):
    lines = hand_lines()
    lines[9] = "not-a-float"
    with pytest.raises(BalFormatError, match=r"malformed float 'not-a-float' in camera parameters") as err:
        read_bal_arrays(write_lines(tmp_path / "a.txt", lines))
    assert err.value.lineno == 10
    lines = hand_lines()
    lines[24] = "nope"
    with pytest.raises(BalFormatError, match="point coordinates") as err:
        read_bal_arrays(write_lines(tmp_path / "b.txt", lines))
    assert err.value.lineno == 25


def test_first_error_in_file_order_wins(tmp_path):
    lines = hand_lines()
    lines[27] = "bad"  # a later error...
    lines[2] = "9 1 3.25 4.5"  # ...and an earlier one
    with pytest.raises(BalFormatError, match="camera index 9") as err:
        read_bal_arrays(write_lines(tmp_path / "a.txt", lines))
    assert err.value.lineno == 3
    # the same across parallel chunks of a large file
    rng = np.random.default_rng(1)
    nc, npt, k = 10, 30000, 80000
    path = tmp_path / "big.txt"
    write_bal_arrays(path, rng.normal(size=(nc, 9)), rng.normal(size=(npt, 3)), rng.integers(0, nc, k),
                     rng.integers(0, npt, k), rng.normal(size=(k, 2)))
    big = path.read_text().split("\n")
    big[70000] = "bad"
    big[5000] = "1 2 3"
    path.write_text("\n".join(big))
    with pytest.raises(BalFormatError, match="observation needs 4 fields, got 3") as err:
        read_bal_arrays(path, n_threads=8)
    assert err.value.lineno == 5001


def test_trailing_content_rejected(tmp_path):
    lines = hand_lines() + ["", "42.0"]
    with pytest.raises(BalFormatError, match="trailing content after point coordinates") as err:
        read_bal_arrays(write_lines(tmp_path / "t.txt", lines))
    assert err.value.lineno == len(hand_lines()) + 1


def test_python_number_syntax(tmp_path):
    """float() / int() accept a sign, underscores between digits, inf/nan."""
    lines = hand_lines()
    lines[1] = "+0 0_0 1_000.5 -inf"
    lines[5] = "nan"
    cams, _, ci, pi, pix = read_bal_arrays(write_lines(tmp_path / "a.txt", lines))
    assert ci[0] == 0 and pi[0] == 0 and pix[0, 0] == 1000.5 and np.isneginf(pix[0, 1])
    assert np.isnan(cams[0, 0])
    lines[1] = "0 0 1__0 2"
    with pytest.raises(BalFormatError, match="malformed observation"):
        read_bal_arrays(write_lines(tmp_path / "b.txt", lines))


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(OSError):
        read_bal_arrays(tmp_path / "nope.txt")


@pytest.mark.gpu
def test_problem_round_trip(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_01941_b200 as P
    from paper_2007_01941_b200.balio import read_bal, write_bal

    prob = P.BundleProblem(*scenes.random_problem(21, n_cameras=4, n_points=12, pixel_noise=0.7).arrays())
    path = tmp_path / "rt.txt"
    write_bal(path, prob)
    back = read_bal(path, loss="huber")
    assert back.loss == "huber"
    assert read_bal(path) == prob
