"""The `fus` command-line front end (build/fus, csrc/fus_cli.cpp) over the drop-in
(reference: tools/fus_cli.cpp). CPU cases: plan output, option handling and exit codes.
GPU cases: the reference's criterion 10 (timings.csv columns and rows, tests/acceptance.cpp:294-330),
manifest.json layout and reload (tools/fus_cli.cpp:49-72,177,318-324), on-axis CSVs equal to the
Python mirror's run_cascade, VIE mode, and the built-in validate suite."""
import json
import os
import subprocess

import pytest

from paper_2011_03009_b200 import fus

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "fus")


def run(*args, cwd=None):
    if not os.path.exists(EXE):
        pytest.fail("build/fus missing: run __graft_entry__.build()")
    p = subprocess.run([EXE, *args], capture_output=True, text=True, cwd=cwd, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_plan_reproduces_the_criterion_5_golden():
    # proj/test_output.txt:31 — H131 water n_w 6: 914x737x737 reference, p2 366x295x295, 15.59x
    rc, out, _ = run("plan", "--transducer", "H131", "--medium", "water", "--harmonics", "5", "--nw", "6")
    assert rc == 0
    assert "reference mesh (harmonic 5): 914 x 737 x 737" in out
    line = next(l for l in out.splitlines() if l.strip().startswith("p2:"))
    assert "366 x 295 x 295" in line and "reduction 15.5868x" in line  # 15.59 to 4 digits
    # the same text as the mirror's plan (host arithmetic, bit-exact)
    t = fus.transducer_preset("H131", 100.0, 4096)
    plan = fus.plan_nested_meshes(t, fus.medium_preset("water"), 10.2e-3, 6, 5)
    assert f"{plan.reference.dims[0]} x {plan.reference.dims[1]} x {plan.reference.dims[2]}" in out


def test_plan_reads_medium_and_transducer_files(tmp_path):
    (tmp_path / "m.cfg").write_text("name = tank\nrho0 = 1000\nc0 = 1480\nbeta = 3.5\nalpha0 = 0.2\neta = 2\n")
    (tmp_path / "t.cfg").write_text("name = bowl\nf0 = 1.1e6\nfocal_length = 35e-3\nouter_radius = 16.5e-3\n"
                                    "n_points = 256\n")
    rc, a, _ = run("plan", "--transducer", str(tmp_path / "t.cfg"), "--medium", str(tmp_path / "m.cfg"),
                   "--harmonics", "5")
    rc2, b, _ = run("plan", "--transducer", "H131", "--medium", "water", "--harmonics", "5")
    assert rc == 0 and rc2 == 0 and a == b  # the files restate the H131 / water presets


@pytest.mark.parametrize("args", [
    (),
    ("frobnicate",),
    ("plan", "--bogus", "1"),
    ("plan", "--nw", "six"),
    ("plan", "--harmonics"),
    ("simulate", "--mode", "fdtd"),
    ("simulate", "--harmonics", "0"),
    ("simulate", "--manifest", "/nonexistent/manifest.json"),
    ("simulate", "--mode", "vie"),  # needs --medium-map
    ("converge", "--study", "bogus"),
    ("validate", "--nw", "4"),
])
def test_configuration_errors_exit_1(args):
    rc, _, err = run(*args)
    assert rc == 1, (args, err)
    assert "config error" in err


def test_runtime_errors_exit_2(tmp_path):
    # a transducer file with a missing key: std::runtime_error from require_double (src/io.cpp)
    (tmp_path / "t.cfg").write_text("name = bowl\nf0 = 1.1e6\n")
    rc, _, err = run("plan", "--transducer", str(tmp_path / "t.cfg"))
    assert rc == 2 and err.startswith("error:")
    # an unknown medium name is read as a config path (tools/fus_cli.cpp:86-88): runtime error too
    rc, _, err = run("plan", "--medium", "unobtainium")
    assert rc == 2 and "cannot open config file 'unobtainium'" in err


def test_help():
    rc, out, _ = run("--help")
    assert rc == 0 and "simulate" in out and "converge" in out


CRIT10 = ["--transducer", "H101", "--medium", "water", "--power", "100", "--f0", "0.2e6", "--harmonics", "5",
          "--nw", "6", "--np", "256"]


@pytest.mark.gpu
def test_criterion_10_timing_table_and_manifest(tmp_path):
    out = tmp_path / "acceptance10_out"
    rc, stdout, err = run("simulate", *CRIT10, "--out", str(out))
    assert rc == 0, err
    lines = (out / "timings.csv").read_text().splitlines()
    assert lines[0] == "harmonic,n_voxels,meshing_s,interpolation_s,evaluate_Gk_s,compute_p_s"
    rows = [[float(c) for c in l.split(",")] for l in lines[1:]]
    assert [int(r[0]) for r in rows] == [2, 3, 4, 5] and all(len(r) == 6 for r in rows)
    vox = [r[1] for r in rows]
    assert vox == sorted(vox)
    assert all(v >= 0 for r in rows for v in r[2:])
    # console table (tools/fus_cli.cpp:123-130)
    head = next(l for l in stdout.splitlines() if l.startswith("p_i"))
    assert head.split() == ["p_i", "N", "voxels", "Meshing", "Interpolation", "Evaluate", "G_ki", "Compute", "p_i"]
    assert "wrote 5 harmonic(s) to" in stdout
    # manifest: nlohmann dump(2) of the RunConfig (sorted keys, 2-space indent)
    text = (out / "manifest.json").read_text()
    m = json.loads(text)
    assert m == {"transducer": "H101", "medium": "water", "power": 100.0, "f0_override": 200000.0,
                 "n_harmonics": 5, "n_w": 6, "d": 0.0102, "n_points": 256, "mode": "homogeneous",
                 "medium_map": "", "out": str(out), "threads": 0, "dump_fields": False, "width_scale": 1.0}
    assert text == json.dumps(m, sort_keys=True, indent=2, separators=(",", ": ")) + "\n"
    for n in range(1, 6):
        assert (out / f"onaxis_p{n}.csv").exists()
    assert (out / "meshplan.txt").read_text().startswith("nested mesh plan (n_w = 6")

    # the on-axis profiles are the mirror's run_cascade + extract_on_axis, digit for digit
    w = fus.medium_preset("water")
    t = fus.transducer_preset("H101", 100.0, 256)
    t.f0 = 0.2e6
    res = fus.run_cascade(fus.CascadeConfig(w, t, fus.plan_nested_meshes(t, w, 10.2e-3, 6, 5), 5))
    for n in (1, 3, 5):
        prof = fus.extract_on_axis(res.p(n))
        fus.write_on_axis_csv(str(tmp_path / f"mirror_p{n}.csv"), prof.x, prof.p)
        assert (tmp_path / f"mirror_p{n}.csv").read_text() == (out / f"onaxis_p{n}.csv").read_text()

    # reload the manifest into a fresh directory: same outputs
    m["out"] = str(tmp_path / "again")
    (tmp_path / "m.json").write_text(json.dumps(m, indent=2))
    rc, _, err = run("simulate", "--manifest", str(tmp_path / "m.json"))
    assert rc == 0, err
    for n in range(1, 6):
        assert (tmp_path / "again" / f"onaxis_p{n}.csv").read_text() == (out / f"onaxis_p{n}.csv").read_text()


@pytest.mark.gpu
def test_simulate_single_harmonic_and_field_dump(tmp_path):
    rc, stdout, err = run("simulate", "--transducer", "H131", "--f0", "0.25e6", "--harmonics", "1", "--np", "128",
                          "--dump-fields", "--out", str(tmp_path / "o"))
    assert rc == 0, err
    assert not (tmp_path / "o" / "timings.csv").exists()  # only written for >= 2 harmonics
    hdr = fus.parse_key_value_file(str(tmp_path / "o" / "p1.bin.hdr"))
    n = int(hdr["nx"]) * int(hdr["ny"]) * int(hdr["nz"])
    assert os.path.getsize(tmp_path / "o" / "p1.bin") == 16 * n


@pytest.mark.gpu
def test_simulate_vie_mode_with_a_slab(tmp_path):
    w = fus.medium_preset("water")
    t = fus.transducer_preset("H131", 100.0, 128)
    t.f0 = 0.25e6
    focus = float(t.focal_length)
    rc, stdout, err = run("simulate", "--transducer", "H131", "--f0", "0.25e6", "--harmonics", "2", "--np", "128",
                          "--mode", "vie", "--medium-map", f"slab:liver:{focus - 5e-3}:4e-3", "--out",
                          str(tmp_path / "v"))
    assert rc == 0, err
    lines = (tmp_path / "v" / "timings.csv").read_text().splitlines()
    assert len(lines) == 2 and lines[1].startswith("2,")
    rc, _, err = run("simulate", "--transducer", "H131", "--f0", "0.25e6", "--harmonics", "2", "--np", "128",
                     "--mode", "vie", "--medium-map", "slab:liver:0.03", "--out", str(tmp_path / "bad"))
    assert rc == 1 and "slab:<medium>" in err


@pytest.mark.gpu
def test_validate_suite_passes():
    rc, out, err = run("validate")
    assert rc == 0, out + err
    assert out.count("[ ok ]") == 5 and out.strip().endswith("all checks passed")


@pytest.mark.gpu
def test_converge_quadrature_study(tmp_path):
    # tools/fus_cli.cpp:191-228 on a small study: convergence.csv columns and the console lines
    rc, out, err = run("converge", "--study", "quadrature", "--transducer", "H131", "--f0", "0.5e6",
                       "--np", "128", "--nw-list", "3", "4", "--nw-ref", "6", "--length", "6e-3",
                       "--width", "2e-3", "--out", str(tmp_path / "c"))
    assert rc == 0, err
    lines = (tmp_path / "c" / "convergence.csv").read_text().splitlines()
    assert lines[0] == "harmonic,n_w,error_percent"
    rows = [[float(x) for x in l.split(",")] for l in lines[1:]]
    assert [r[1] for r in rows] == [3.0, 4.0] and all(r[2] >= 0 for r in rows)
    assert "fitted log-log slope:" in out and out.count("error =") == 2
