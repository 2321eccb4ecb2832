"""The reference's problem JSON (problem.py:318-389) and the binary stack
form: files written by the REAL reference's rapdb.problem.save
(tests/golden/problem_*.json, tests/golden/make_json_golden.py) load into the
same arrays and re-serialise byte for byte."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_29291_b200 import problem
from paper_2605_29291_b200.errors import ConfigurationError, InputError

FILES = ["problem_rq.json", "problem_eqqp.json", "problem_kml.json"]


@pytest.mark.parametrize("name", FILES)
def test_load_reference_json_and_roundtrip(name, tmp_path):
    path = os.path.join(GOLDEN, name)
    raw = json.load(open(path))
    inst = problem.load(path, validate=False)
    n = raw["n"]
    assert (inst.n, inst.m, inst.p) == (raw["n"], raw["m"], raw["p"])
    for i, M in enumerate(raw["Q"]):
        ref = (np.zeros((n, n)) if isinstance(M, dict) and not M["data"] else
               problem._matrix_from_json(M, (n, n)))
        np.testing.assert_array_equal(inst.Q[i], ref)
    np.testing.assert_array_equal(inst.q, np.array(raw["q"]))
    np.testing.assert_array_equal(inst.primal_set.lower, np.array(raw["primal_set"]["lower"]))
    out = tmp_path / "out.json"
    problem.save(inst, str(out))
    assert out.read_text() == open(path).read()


def test_binary_stack_roundtrip(tmp_path):
    inst = problem.load(os.path.join(GOLDEN, "problem_eqqp.json"))
    p = str(tmp_path / "s.npz")
    problem.save_stack(inst, p)
    back = problem.load_stack(p)
    np.testing.assert_array_equal(back.Q, inst.Q)
    np.testing.assert_array_equal(back.A, inst.A)
    assert back.p == inst.p and back.name == inst.name


def test_unsupported_descriptors():
    base = json.load(open(os.path.join(GOLDEN, "problem_rq.json")))
    d = dict(base, primal_set={"type": "simplex", "dim": base["n"], "scale": 1.0})
    with pytest.raises(ConfigurationError):
        problem.from_json_dict(d)
    d = dict(base, cone={"type": "soc", "dim": base["m"]})
    with pytest.raises(ConfigurationError):
        problem.from_json_dict(d)
    d = dict(base, primal_set={"type": "what"})
    with pytest.raises(InputError):
        problem.from_json_dict(d)
    d = dict(base)
    del d["Q"]
    with pytest.raises(InputError):
        problem.from_json_dict(d)
