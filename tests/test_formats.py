"""Wire/disk formats: history CSV (stk/report.hpp:22-26), result CSV
(stk/bench.hpp:210-242), MatrixMarket (stk/matrix_market.hpp:16-80).  CPU only."""
import io

import numpy as np
import pytest

from conftest import ROOT  # noqa: F401


def test_history_csv(stk):
    from paper_1912_10082_b200 import formats
    buf = io.StringIO()
    formats.write_history_csv(buf, [0.5, 1e-5, 1.234567891e-9, 100000.0, 1e6])
    assert buf.getvalue() == "iter,relres\n1,0.5\n2,1e-05\n3,1.23457e-09\n4,100000\n5,1e+06\n"


def test_result_csv(stk):
    from paper_1912_10082_b200 import formats
    rows = [formats.ResultRow("rksm", 199, 100, 14, 15, 9, 0.123456, 3.2e-9, 1.5e-7),
            formats.ResultRow("cn", 199, 100, 0, 0, 0, 2.0, 0.0)]
    buf = io.StringIO()
    formats.write_result_csv(buf, rows)
    assert buf.getvalue() == (
        "method,N_h,N_t,iters,mu_mem,rank,time_s,relres,err_oracle\n"
        "rksm,199,100,14,15,9,0.1235,3.200000e-09,1.500000e-07\n"
        "cn,199,100,0,0,0,2.0000,0.000000e+00,\n")
    buf = io.StringIO()
    formats.write_result_csv(buf, rows[:1], stable_time=True)
    assert ",0.0000," in buf.getvalue()  # byte-stable reruns


def test_matrix_market_roundtrip_fem_and_bands(stk):
    from paper_1912_10082_b200 import assembly, formats
    m, a = assembly.fem1d_matrices(assembly.SpaceGrid1D(0.0, 1.0, 5))
    tm = formats.tridiagonal_triplets(m)
    buf = io.StringIO()
    formats.write_matrix_market(buf, tm)
    text = buf.getvalue()
    lines = text.splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real symmetric"
    assert lines[1] == "5 5 9"  # lower triangle only
    i, j, v = lines[2].split()
    assert (i, j) == ("1", "1") and float(v) == m.diag[0] and v == format(float(m.diag[0]), ".17g")
    back = formats.read_matrix_market(io.StringIO(text))
    assert back.symmetric and np.array_equal(back.dense(), m.dense())
    d, c = assembly.heat_time_matrices(assembly.TimeGrid(4, 1.0))
    buf = io.StringIO()
    formats.write_matrix_market(buf, formats.bidiagonal_triplets(d))
    assert buf.getvalue().splitlines()[0].endswith("general")
    assert np.array_equal(formats.read_matrix_market(io.StringIO(buf.getvalue())).dense(),
                          d.dense())
    ws = assembly.wave_space_matrices(assembly.SpaceGrid1D(0.0, 1.0, 12))
    for band in (ws.M, ws.A):
        buf = io.StringIO()
        formats.write_matrix_market(buf, formats.band7_triplets(band))
        assert np.array_equal(formats.read_matrix_market(io.StringIO(buf.getvalue())).dense(),
                              band.dense())


@pytest.mark.parametrize("text,msg", [
    ("", "empty input"),
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", "unsupported header"),
    ("%%MatrixMarket matrix coordinate real general\n% c\nx y\n", "bad size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "truncated"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n", "duplicate"),
])
def test_matrix_market_errors(stk, text, msg):
    from paper_1912_10082_b200 import formats
    from paper_1912_10082_b200.errors import ArgumentError
    with pytest.raises(ArgumentError, match=msg):
        formats.read_matrix_market(io.StringIO(text))


def test_matrix_market_comments_and_symmetric_mirror(stk):
    from paper_1912_10082_b200 import formats
    text = ("%%MatrixMarket matrix coordinate real symmetric\n% comment\n%another\n3 3 3\n"
            "1 1 2.0\n2 1 -1.0\n3 3 4.0\n")
    m = formats.read_matrix_market(io.StringIO(text))
    np.testing.assert_array_equal(m.dense(), [[2, -1, 0], [-1, 0, 0], [0, 0, 4]])
