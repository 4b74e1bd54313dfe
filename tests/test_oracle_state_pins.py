"""Pins of the oracle's VMS stabilisation (reading A-14) and Cahn-Hilliard state
(reading A-10) to independently computed values (tests/state_pins.py), and proof that
the pins have teeth: seeded mutations of exactly those formulas in a copy of oracle.c each
make them fail (the mutated library is loaded in a subprocess through IGA_ORACLE_SO_OVERRIDE).
"""
import os
import subprocess
import sys

import pytest

import state_pins

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")


def test_vms_tau_pinned():
    state_pins.check_vms_tau()


def test_cahn_hilliard_state_pinned():
    state_pins.check_ch_state()


# (pin, original text in oracle.c, mutated text): plausible mistakes in the readings
MUTATIONS = [
    ("vms", "D[k][i] = 2.0 / Q->hpar[k] * Q->dxi_dx[k][i];", "D[k][i] = 1.0 / Q->hpar[k] * Q->dxi_dx[k][i];"),  # 2/h -> 1/h
    ("vms", "+ uGu + CI * nu * nu * GG);", "+ uGu);"),                                                  # drop C_I term
    ("vms", "Ct / (dt * dt) + uGu", "Ct / dt + uGu"),                                                   # dt^2 -> dt
    ("vms", "P->tauC = 1.0 / (P->tauM * gg);", "P->tauC = 1.0 / (P->tauM * sqrt(gg));"),               # g.g -> |g|
    ("vms", "uGu += ftau->u[i] * G[i][j] * ftau->u[j];", "uGu += ftau->u[i] * G[i][j];"),              # u.Gu -> sum Gu
    ("vms", "for (int i = 0; i < 3; i++) P->up[i] = -P->tauM * P->rM[i];",
     "for (int i = 0; i < 3; i++) P->up[i] = P->tauM * P->rM[i];"),                                     # sign of u'
    ("ch", "P->M = c * (1.0 - c);", "P->M = c * (1.0 + c);"),
    ("ch", "P->mup = 3.0 * al * (1.0 / (2.0 * th * c * (1.0 - c)) - 2.0);",
     "P->mup = 3.0 * al * (1.0 / (th * c * (1.0 - c)) - 2.0);"),                                       # 2 theta -> theta
    ("ch", "P->mup = 3.0 * al * (1.0 / (2.0 * th * c * (1.0 - c)) - 2.0);",
     "P->mup = 3.0 * al * (1.0 / (2.0 * th * c * (1.0 - c)) - 1.0);"),                                 # -2 -> -1
]


def _build_mutant(tmp_path, orig, new, tag):
    src = open(SRC).read()
    assert src.count(orig) == 1, f"mutation anchor not unique / missing: {orig!r}"
    path = tmp_path / f"mut_{tag}.c"
    path.write_text(src.replace(orig, new))
    so = tmp_path / f"libmut_{tag}.so"
    subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                           "-o", str(so), str(path), "-lm"])
    return str(so)


def _run_pin(which, so=None):
    env = dict(os.environ)
    if so:
        env["IGA_ORACLE_SO_OVERRIDE"] = so
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests")])
    return subprocess.run([sys.executable, os.path.join(ROOT, "tests", "state_pins.py"), which], env=env,
                          capture_output=True, text=True, timeout=600)


def test_pins_pass_in_subprocess():
    for which in ("vms", "ch"):
        r = _run_pin(which)
        assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.parametrize("k", range(len(MUTATIONS)))
def test_mutated_oracle_fails_pins(tmp_path, k):
    which, orig, new = MUTATIONS[k]
    so = _build_mutant(tmp_path, orig, new, str(k))
    r = _run_pin(which, so)
    assert r.returncode != 0, f"mutation {k} ({new!r}) was NOT caught by the {which} pins"
    assert "AssertionError" in r.stderr, r.stderr[-2000:]
