"""File formats of the drop-in (include/fus/io.hpp contracts, tests/test_io.cpp cases) through the
Python mirror, and agreement with the C++ shim's writers (run through build/test_fus_api in
test_abi). CPU only."""
import numpy as np
import pytest

from paper_2011_03009_b200 import fus


def test_key_value_parser(tmp_path):
    p = tmp_path / "kv.txt"
    p.write_text("# comment\n\n  key1 = 7.5  \nkey2=text value\n")
    kv = fus.parse_key_value_file(str(p))
    assert kv == {"key1": "7.5", "key2": "text value"}
    assert fus.require_double(kv, "key1", "t") == 7.5 and fus.require_string(kv, "key2", "t") == "text value"
    with pytest.raises(RuntimeError):
        fus.require_double(kv, "missing", "t")
    with pytest.raises(RuntimeError):
        fus.require_double(kv, "key2", "t")
    (tmp_path / "bad.txt").write_text("ok = 1\nno equals sign here\n")
    with pytest.raises(RuntimeError, match=":2:"):
        fus.parse_key_value_file(str(tmp_path / "bad.txt"))
    with pytest.raises(RuntimeError):
        fus.parse_key_value_file(str(tmp_path / "nope.txt"))


def test_csv_writers(tmp_path):
    fus.write_on_axis_csv(str(tmp_path / "a.csv"), [0.01, 0.02], [3 + 4j, 1])
    lines = (tmp_path / "a.csv").read_text().splitlines()
    assert lines[0] == "x_m,re_Pa,im_Pa,abs_Pa" and lines[1].startswith("0.01,") and ",5" in lines[1]
    fus.write_csv(str(tmp_path / "g.csv"), ["a", "b"], [[1, 2], [3, 4.5]])
    assert (tmp_path / "g.csv").read_text().splitlines() == ["a,b", "1,2", "3,4.5"]


def test_field_dump_and_medium_map_round_trip(tmp_path):
    g = fus.make_grid([0, 0, 0], [3e-4, 2e-4, 2e-4], 1e-4, 2)
    k = fus.complex_wavenumber(fus.medium_preset("water"), 1.1e6, 2)
    v = fus.random_vector(g.count(), 3)
    fus.write_field_dump(str(tmp_path / "f.bin"), fus.HarmonicField(g, v, k))
    hdr = fus.parse_key_value_file(str(tmp_path / "f.bin.hdr"))
    assert fus.require_double(hdr, "nx", "h") == g.dims[0] and fus.require_double(hdr, "dx", "h") == g.dx
    assert fus.require_double(hdr, "k_re", "h") == k.k.real and hdr["layout"] == "x_fastest_complex_f64_le"
    assert np.array_equal(np.fromfile(tmp_path / "f.bin", "<c16"), v)
    g = fus.make_grid([0, 0, 0], [5e-3, 4e-3, 3e-3], 1e-3, 1)
    m = fus.slab_map(g, fus.medium_preset("water"), fus.medium_preset("liver"), 2e-3, 2e-3)
    fus.write_medium_map(str(tmp_path / "m.hdr"), str(tmp_path / "m.bin"), m)
    back = fus.load_medium_map(str(tmp_path / "m.hdr"), fus.medium_preset("water"))
    assert back.grid.dims == g.dims and back.grid.dx == g.dx
    assert np.array_equal(back.c, m.c) and np.array_equal(back.beta, m.beta)
    (tmp_path / "m.bin").write_bytes((tmp_path / "m.bin").read_bytes()[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        fus.load_medium_map(str(tmp_path / "m.hdr"), fus.medium_preset("water"))
