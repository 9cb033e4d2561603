"""The reference's own verification battery (tmd::run_verification,
proj/src/verify.cpp:822-845) run against the B200 path: oracle/_ref/refverify_b200
links the unmodified reference sources with integration/potential_b200.cpp,
which replaces tmd::evaluate_forces, so every evaluate_forces call of the
battery — scheme/width equivalence, Newton, filter soundness, precision gap,
determinism and a 25-step Engine rerun — runs on the GPU.

Expected non-passes, asserted precisely:
  * kmax_sweep: only its bitwise clauses ("v3 k_max=0 not bitwise", "v3
    k_max=16 differs from cached scalar path") — bit equality with the CPU's
    glibc libm is out of reach for any GPU path; its tolerance
    sweep (1e-12 E, 1e-10 F) must pass;
  * zeta_gradients on the SiC table: the check exercises the reference's own
    scalar kern::zeta_term against finite differences (no evaluate_forces
    call), which misses its 1e-6 gate for SiC's c^2/d^2 = 3.8e7 — a property
    of the reference, not of this path.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "refverify_b200")
BITWISE_NOTES = {"v3 k_max=0 not bitwise", "v3 k_max=16 differs from cached scalar path"}


def _run(*args):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/refverify_b200 not built (needs /root/reference at build time)")
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    rows = {}
    for line in p.stdout.splitlines():
        status, name, *detail = line.split(" ", 2)
        rows[name] = (status, detail[0] if detail else "")
    assert rows, p.stdout + p.stderr
    return rows


def _check(rows, allowed_fail=()):
    assert len(rows) == 16
    for name, (status, detail) in rows.items():
        if name == "kmax_sweep" and status == "FAIL":
            notes = {x.strip() for x in detail.split(";") if x.strip()}
            assert notes <= BITWISE_NOTES, detail
        elif name in allowed_fail:
            continue
        else:
            assert status == "PASS", (name, detail)


def test_reference_battery_silicon():
    rows = _run()
    _check(rows)
    # the GPU path's scheme/width sweep against compute_ref, as the battery measures it
    assert rows["scheme_equivalence"][0] == "PASS"
    assert rows["determinism"][0] == "PASS"


def test_reference_battery_sic():
    _check(_run(os.path.join(ROOT, "tests", "golden", "SiC.tersoff")),
           allowed_fail=("zeta_gradients",))


ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.parametrize("criterion", range(1, 9))
def test_reference_acceptance_gate(criterion):
    """proj/tests/acceptance.cpp criteria 1-8 with evaluate_forces on the B200
    (1: single-precision 10^4-step trajectory within 2e-5 of double; 2: every
    scheme x width x k_max within 1e-12 E / 1e-10 F of compute_ref; 4: 10^4-step
    NVE — drift < 1e-4, |sum F| < 1e-10, momentum < 1e-8; 5: filter on/off
    1e-12; 3, 6, 7 are CPU-side; 8 reports ns/day, non-gating)."""
    if not os.path.exists(ACC):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")
    p = subprocess.run([ACC, str(criterion)], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0 and p.stdout.startswith("PASS"), p.stdout + p.stderr


def test_engine_run_through_the_drop_in():
    """tmd::Engine::run (engine.cpp:174-199) on cfg 2 with the B200 drop-in as
    evaluate_forces follows the stock CPU Engine: same rebuild schedule, Etot
    within 1e-9 relative after 100 steps (oracle/engine_run_main.cpp)."""
    import json
    b200 = os.path.join(ROOT, "oracle", "_ref", "engine_run_b200")
    cpu = os.path.join(ROOT, "oracle", "_ref", "engine_run_cpu")
    if not (os.path.exists(b200) and os.path.exists(cpu)):
        pytest.skip("oracle/_ref/engine_run_* not built (needs /root/reference at build time)")
    rg = json.loads(subprocess.run([b200, "100"], capture_output=True, text=True,
                                   timeout=600).stdout)
    rc = json.loads(subprocess.run([cpu, "100"], capture_output=True, text=True,
                                   timeout=600).stdout)
    assert rg["rebuilds"] == rc["rebuilds"] == 4
    assert abs(rg["etot_first"] - rc["etot_first"]) <= 1e-12 * abs(rc["etot_first"])
    assert abs(rg["etot_last"] - rc["etot_last"]) <= 1e-9 * abs(rc["etot_last"])
