"""Host-side logic of the product, no GPU (CPU suite).

* the C-ABI library loads and exports every symbol include/tersoff_b200.h declares;
* the parameter parser mirrors proj/src/params.cpp (grammar, interning,
  validation messages, round-trip serialization), checked against the oracle's
  independent restatement and the reference itself when present;
* the generators are bit-identical to the reference's (engine.cpp:28-116,
  verify.cpp:83-104);
* evaluate_forces option validation mirrors potential_opt.cpp:51-138;
* without a GPU, device entry points fail with an error code, never a crash.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.oracle import SI_TEXT, parse_param_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol(tb):
    from paper_1607_02904_b200 import _lib
    header = open(os.path.join(ROOT, "include", "tersoff_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tsf_\w+)\s*\(", header, re.M))
    assert len(declared) >= 35
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert {p[0] for p in _lib.PROTOTYPES} == declared
    lib.tsf_version.restype = C.c_char_p
    assert b"sm_100a" in lib.tsf_version()


def test_builtin_silicon_and_round_trip(tb):
    p = tb.builtin_silicon()
    assert p.species_count == 1 and p.species_names == ["Si"] and p.r_cut_max == 3.2
    text = p.serialize()
    assert text.startswith("# element1 element2 element3")
    q = tb.parse_params(text)
    assert q.serialize() == text
    np.testing.assert_array_equal(p.rows, parse_param_text(SI_TEXT).rows)


def test_sic_table(tb):
    text = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
    p = tb.parse_params(text)
    assert p.species_names == ["Si", "C"] and p.r_cut_max == 3.0
    assert p.species_id("C") == 1 and p.species_id("Ge") == -1
    np.testing.assert_array_equal(p.rows, parse_param_text(text).rows)


def test_lammps_style_cross_rows(tb):
    """LAMMPS-format tables (n = beta = 0 on cross rows (i, j, k), j != k,
    whose bond-order fields are never read) parse; a zero eta on an
    (i, j, j) row is still refused, as the reference refuses it."""
    import systems
    text = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
    lmp = systems.lammps_style(text)
    assert lmp != text
    p, q = tb.parse_params(lmp), tb.parse_params(text)
    assert p.species_names == q.species_names and p.r_cut_max == q.r_cut_max
    bad = lmp.replace("C  Si Si 3.0 1.0 0.0 3.8049e4 4.3484 -0.57058 0.72751",
                      "C  Si Si 3.0 1.0 0.0 3.8049e4 4.3484 -0.57058 0.0")
    assert bad != lmp
    with pytest.raises(tb.ParseError) as exc:
        tb.parse_params(bad)
    assert "'eta' must be positive" in str(exc.value)


@pytest.mark.parametrize("text,needle", [
    ("", "no entries found"),
    ("Si Si Si 1 2 3", "truncated entry"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 x", "expected a number"),
    ("Si Si Si 2.5 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 3264", "must be an integer"),
    ("Si Si Si 2 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 3264", "must be 1 or 3"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.0 3.2 3264", "'D' must be positive"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 0.1 0.2 3.2 3264", "'R' must exceed D"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 0 0.3 1.3 95.3 3.0 0.2 3.2 3264", "'eta' must be positive"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 -0.3 1.3 95.3 3.0 0.2 3.2 3264", "'beta' must be non-negative"),
    ("Si Si Si 3 1 1.3 4.8 0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 3264", "'d' must be nonzero"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 -1", "'A' must be non-negative"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 -95.3 3.0 0.2 3.2 3264", "'B' must be non-negative"),
    ("Si Si Si 3 -1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 3264", "'gamma' must be"),
    ("Si Si Si 3 1 1.3 4.8 2.0 0 22.9 0.3 1.3 95.3 3.0 0.2 3.2 inf", "not finite"),
    (SI_TEXT + SI_TEXT, "duplicate entry"),
    (SI_TEXT + SI_TEXT.replace("Si Si Si", "Si C Si"), "missing entry"),
])
def test_parse_errors(tb, text, needle):
    with pytest.raises(tb.ParseError) as exc:
        tb.parse_params(text)
    assert needle in str(exc.value)


def test_comments_and_wrapping(tb):
    text = ("# header\nSi Si Si 3.0 1.0 1.3258 4.8381   # trailing\n 2.0417 0.0000 22.956\n"
            "0.33675 1.3258 95.373 3.0 0.2\n3.2394 3264.7\n")
    assert tb.parse_params(text).serialize() == tb.builtin_silicon().serialize()


def test_load_params_errors(tb, tmp_path):
    with pytest.raises(tb.ConfigError):
        tb.load_params("/nonexistent/file.tersoff")
    f = tmp_path / "Si.tersoff"
    f.write_text(SI_TEXT)
    assert tb.load_params(str(f)).serialize() == tb.builtin_silicon().serialize()


def test_generators_match_reference(tb, reference):
    R = reference
    rp = R.params(SI_TEXT)
    for cells, jit, seed in [(2, 0.12, 722), (4, 0.12, 32), (3, 0.35, 5)]:
        s = tb.perturbed_lattice(tb.builtin_silicon(), cells, jit, seed)
        xyz, _, sp, box, _ = R.system_arrays(R.perturbed_lattice(rp, cells, jit, seed))
        assert np.array_equal(s.positions, xyz) and np.array_equal(s.species, sp)
        assert np.array_equal(s.box.lengths, box)
    for T, seed in [(300.0, 7), (1600.0, 12345), (0.0, 3)]:
        s = tb.make_diamond_lattice(3, 2, 4)
        tb.init_velocities(s, T, seed)
        h = R.diamond_lattice(3, 2, 4)
        R.init_velocities(h, T, seed)
        xyz, vel, *_ = R.system_arrays(h)
        assert np.array_equal(s.positions, xyz) and np.array_equal(s.velocities, vel)


def test_thermo_helpers(tb):
    s = tb.make_diamond_lattice(2, 2, 2)
    tb.init_velocities(s, 300.0, 7)
    assert abs(tb.temperature(s) - 300.0) <= 1e-9
    assert max(abs(p) for p in tb.total_momentum(s)) < 1e-10
    with pytest.raises(tb.ConfigError):
        tb.make_diamond_lattice(0, 1, 1)
    with pytest.raises(tb.ConfigError):
        tb.init_velocities(s, -1.0, 1)


def test_option_validation():
    from paper_1607_02904_b200.api import _resolve_options, ConfigError
    assert _resolve_options("auto", "opt-d", 0, 16, 1) == 0
    assert _resolve_options("v2", "mixed", 8, 16, 4) == 1
    assert _resolve_options("v1", "single", 4, 0, 1) == 2
    for bad in [("v9", "opt-d", 0, 16, 1), ("auto", "quad", 0, 16, 1), ("auto", "opt-d", 3, 16, 1),
                ("auto", "opt-d", 0, -1, 1), ("auto", "opt-d", 0, 16, 0),
                ("ref", "single", 0, 16, 1), ("scalar-opt", "mixed", 0, 16, 1)]:
        with pytest.raises(ConfigError):
            _resolve_options(*bad)


def test_device_calls_fail_cleanly_without_gpu(tb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((tb.CudaError, tb.ConfigError)):
        tb.Context(tb.builtin_silicon(), 0)


def test_bench_algorithmic_work_counter(tb, oracle):
    """bench.py's P/T counts (ALGO_FLOP = 75 P + 143 T) vs a direct loop."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    import systems
    sic = open(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")).read()
    for c in [systems.liquid_like(tb, 3, 0.35, 5), systems.zincblende(tb, sic, 3, jitter=0.1)]:
        op = parse_param_text(c.params_text)
        off, nb = oracle.build_neighbor_list(c.xyz, c.box, c.periodic, op.r_cut_max, c.skin)
        so, sn = oracle.filter(c.xyz, c.box, c.periodic, off, nb, op.r_cut_max)
        P, T = bench.algorithmic_work(c.xyz, c.species, c.box, so, sn, op.rows, op.ns)
        Pb = Tb = 0
        for i in range(len(so) - 1):
            seg = sn[so[i]:so[i + 1]]

            def r2(a, b):
                d = c.xyz[b] - c.xyz[a]
                d -= c.box * np.floor(d / c.box + 0.5)
                return d @ d
            for j in seg:
                si, sj = c.species[i], c.species[j]
                if r2(i, j) > op.rows[(si * op.ns + sj) * op.ns + sj, 15]:
                    continue
                Pb += 1
                Tb += sum(1 for k in seg if k != j and
                          r2(i, k) <= op.rows[(si * op.ns + sj) * op.ns + c.species[k], 15])
        assert (P, T) == (Pb, Tb)


def test_snapshot_round_trip(tb, sic_text, tmp_path):
    """TSFSNAP1 (csrc/tsf_snapshot.cpp): the product's writer and reader, the
    independent numpy reader (oracle/snapshot.py) and hashlib agree; float64
    coordinates round-trip bit for bit, float32 ones as the float32 rounding."""
    import hashlib
    from oracle import snapshot as osnap
    params = tb.parse_params(sic_text)
    s = tb.perturbed_lattice(params, 3, 0.2, 7)
    tb.init_velocities(s, 900.0, 5)
    for f32, vel in [(False, False), (False, True), (True, False), (True, True)]:
        path = str(tmp_path / f"s_{int(f32)}{int(vel)}.tsfsnap")
        sha = tb.save_snapshot(path, s, float32_coords=f32, velocities=vel)
        raw = open(path, "rb").read()
        assert hashlib.sha256(raw[:-32]).hexdigest() == sha == raw[-32:].hex()
        info = tb.snapshot_info(path)
        assert info["natoms"] == s.natoms and info["species_count"] == 2
        assert info["sha256"] == sha
        back = tb.load_snapshot(path)
        ref = osnap.read(path)
        want = s.positions.astype(np.float32).astype(np.float64) if f32 else s.positions
        assert np.array_equal(back.positions, want) and np.array_equal(ref["positions"], want)
        assert np.array_equal(back.species, s.species) and np.array_equal(ref["species"],
                                                                            s.species)
        assert back.species_masses == list(s.species_masses)
        assert np.array_equal(back.box.lengths, s.box.lengths)
        assert np.array_equal(ref["box"], s.box.lengths)
        assert np.array_equal(back.box.periodic, s.box.periodic)
        if vel:
            assert np.array_equal(back.velocities, s.velocities)
            assert np.array_equal(ref["velocities"], s.velocities)
        else:
            assert not back.velocities.any() and ref["velocities"] is None
    # a flipped byte anywhere fails the checksum in both readers
    bad = bytearray(open(path, "rb").read())
    bad[100] ^= 1
    badp = str(tmp_path / "bad.tsfsnap")
    open(badp, "wb").write(bytes(bad))
    with pytest.raises(tb.ConfigError, match="SHA-256"):
        tb.load_snapshot(badp)
    with pytest.raises(ValueError, match="SHA-256"):
        osnap.read(badp)
    with pytest.raises(tb.ConfigError, match="cannot open"):
        tb.load_snapshot(str(tmp_path / "missing.tsfsnap"))
    s.species[3] = 5
    with pytest.raises(tb.ConfigError, match="species id"):
        tb.save_snapshot(str(tmp_path / "x.tsfsnap"), s)


def test_bench_reference_arm_inputs_without_product(tb, reference):
    """bench.py --impl reference builds the workload through the reference's own
    generator (oracle/_ref) and never loads the product; its arrays equal the
    GPU arm's (bench.make_system) bit for bit."""
    import subprocess
    import sys
    import bench
    from oracle.oracle import Reference
    for cfg in ("si32k", "sic256k"):
        a = bench.make_system(cfg)
        b = bench.make_system_reference(cfg, Reference())
        for x, y in zip(a[1:5], b[1:5]):
            assert np.array_equal(np.asarray(x), np.asarray(y)), cfg
        assert a[5] == b[5]
        assert tb.parse_params(a[0]).serialize() == tb.parse_params(b[0]).serialize()
    code = ("import sys, bench; from oracle.oracle import Reference; "
            "bench.make_system_reference('si32k', Reference()); "
            "assert not [m for m in sys.modules if m.startswith('paper_1607_02904_b200')]")
    subprocess.run([sys.executable, "-c", code], cwd=ROOT, check=True)
