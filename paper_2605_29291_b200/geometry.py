"""Primal sets, cones and dual balls: host-side *descriptors* for the device path.

Mirrors the reference's geometry surface (``pkg/src/rapdb/geometry.py``) for the
objects the hot path uses:

* ``Box`` (``geometry.py:31-47``) -- the primal set; projected on device by the
  fused primal-step kernel (clip against per-coordinate ``lower``/``upper``,
  infinite bounds allowed).
* ``NonnegOrthant`` (``geometry.py:170-178``) -- the constraint cone; its dual
  projection ``max(lam, 0)`` runs on device inside the dual-momentum phase.
* ``Unbounded`` / ``JointBall`` / ``SplitBall`` (``geometry.py:263-311``) -- the
  optional dual-norm ball, a radial rescale applied after the cone projection.

The small host ``project`` helpers below exist for API compatibility (users call
them on single points, e.g. ``initial_iterate``); the solver never routes its
iterations through them.  Sets/cones the device path does not build (SOC,
product cones, balls/simplices as primal sets) are rejected with
``ConfigurationError`` when a solve is attempted, not computed on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

from .errors import ConfigurationError, InputError

__all__ = [
    "Box", "NonnegOrthant", "Unbounded", "JointBall", "SplitBall",
    "SimpleSet", "Cone", "DualBall", "project_set", "project_dual_cone",
    "bregman_p", "bregman_d", "set_dim", "cone_dim", "ball_code",
]


@dataclass(frozen=True)
class Box:
    lower: np.ndarray
    upper: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lower, dtype=float)
        hi = np.asarray(self.upper, dtype=float)
        object.__setattr__(self, "lower", lo)
        object.__setattr__(self, "upper", hi)
        if lo.shape != hi.shape or lo.ndim != 1:
            raise InputError("box bounds must be 1-d arrays of equal length")
        if np.any(lo > hi):
            raise InputError("box has lower > upper")

    def project(self, w):
        return np.clip(w, self.lower, self.upper)


@dataclass(frozen=True)
class NonnegOrthant:
    dim: int

    def project(self, w):
        return np.maximum(w, 0.0)

    def project_dual(self, w):
        return np.maximum(w, 0.0)


@dataclass(frozen=True)
class Unbounded:
    def project(self, v, lam):
        return v, lam

    def contains(self, v, lam, tol=0.0):
        return True


@dataclass(frozen=True)
class JointBall:
    radius: float

    def __post_init__(self):
        if self.radius <= 0:
            raise InputError("ball radius must be positive")

    def project(self, v, lam):
        nrm = np.sqrt(v @ v + lam @ lam)
        if nrm <= self.radius:
            return v, lam
        s = self.radius / nrm
        return s * v, s * lam

    def contains(self, v, lam, tol=0.0):
        return np.sqrt(v @ v + lam @ lam) <= self.radius + tol


@dataclass(frozen=True)
class SplitBall:
    radius_v: float
    radius_lam: float

    def __post_init__(self):
        if self.radius_v <= 0 or self.radius_lam <= 0:
            raise InputError("ball radii must be positive")

    def project(self, v, lam):
        nv = np.linalg.norm(v)
        if nv > self.radius_v:
            v = (self.radius_v / nv) * v
        nl = np.linalg.norm(lam)
        if nl > self.radius_lam:
            lam = (self.radius_lam / nl) * lam
        return v, lam

    def contains(self, v, lam, tol=0.0):
        return (np.linalg.norm(v) <= self.radius_v + tol
                and np.linalg.norm(lam) <= self.radius_lam + tol)


class _OutOfScope:
    """Sets and cones of the reference that no BASELINE config uses (SURVEY.md
    section 8: out of scope).  They import, so drop-in code keeps loading, and
    constructing one fails loudly."""

    kind = ""

    def __init__(self, *args, **kwargs):
        raise ConfigurationError(f"{self.kind} (reference geometry.py) is not built on the device path")


class Ball(_OutOfScope):
    kind = "Ball primal set"


class Simplex(_OutOfScope):
    kind = "Simplex primal set"


class NonnegWithLinearEq(_OutOfScope):
    kind = "NonnegWithLinearEq primal set"


class SecondOrderCone(_OutOfScope):
    kind = "SecondOrderCone"


class ProductCone(_OutOfScope):
    kind = "ProductCone"


SimpleSet = Box
Cone = NonnegOrthant
DualBall = Union[Unbounded, JointBall, SplitBall]


def set_dim(s) -> int:
    if isinstance(s, Box):
        return len(s.lower)
    raise ConfigurationError(f"primal set {type(s).__name__} is not supported by the device path")


def cone_dim(c) -> int:
    if isinstance(c, NonnegOrthant):
        return c.dim
    raise ConfigurationError(f"cone {type(c).__name__} is not supported by the device path")


def project_set(s, w):
    w = np.asarray(w, dtype=float)
    if w.shape != (set_dim(s),):
        raise InputError(f"point of dim {w.shape} does not match set of dim {set_dim(s)}")
    return s.project(w)


def project_dual_cone(c, w):
    w = np.asarray(w, dtype=float)
    if w.shape != (cone_dim(c),):
        raise InputError(f"point of dim {w.shape} does not match cone of dim {cone_dim(c)}")
    return c.project_dual(w)


def bregman_p(x, xbar):
    d = np.asarray(x, dtype=float) - np.asarray(xbar, dtype=float)
    return 0.5 * float(d @ d)


bregman_d = bregman_p


def bregman(x, xbar):
    """geometry.py:357-361 (Euclidean generator)."""
    return bregman_p(x, xbar)


def project_dual_ball(d, y):
    """geometry.py:317-320: y = (v, lam) through the dual ball."""
    return d.project(*y) if isinstance(y, tuple) else d.project(y[0], y[1])


def validate_dual_ball(cone, ball):
    """geometry.py:331-335: balls are fine for the orthant (no SOC here)."""
    cone_dim(cone)
    return ball


def ball_code(ball):
    """(kind, r1, r2) triple consumed by ``rapdb_set_params`` (0/1/2 = none/joint/split)."""
    if ball is None or isinstance(ball, Unbounded):
        return 0, 0.0, 0.0
    if isinstance(ball, JointBall):
        return 1, float(ball.radius), 0.0
    if isinstance(ball, SplitBall):
        return 2, float(ball.radius_v), float(ball.radius_lam)
    raise ConfigurationError(f"dual ball {type(ball).__name__} is not supported")


# ---- JSON descriptors (geometry.py:376-421 of the reference) --------------
def set_to_json(s) -> dict:
    if isinstance(s, Box):
        return {"type": "box", "lower": list(s.lower), "upper": list(s.upper)}
    from .errors import ConfigurationError
    raise ConfigurationError(f"primal set {type(s).__name__} is not built on the device path")


def set_from_json(d: dict):
    from .errors import ConfigurationError, InputError
    try:
        kind = d["type"]
        if kind == "box":
            return Box(np.asarray(d["lower"], float), np.asarray(d["upper"], float))
    except (KeyError, TypeError) as exc:
        raise InputError(f"bad set descriptor {d!r}: {exc}") from exc
    if kind in ("ball", "simplex", "nonneg_lineq"):
        raise ConfigurationError(f"primal set type {kind!r} is not built on the device path")
    raise InputError(f"unknown set type {kind!r}")


def cone_to_json(c) -> dict:
    if isinstance(c, NonnegOrthant):
        return {"type": "orthant", "dim": c.dim}
    from .errors import ConfigurationError
    raise ConfigurationError(f"cone {type(c).__name__} is not built on the device path")


def cone_from_json(d: dict):
    from .errors import ConfigurationError, InputError
    try:
        kind = d["type"]
        if kind == "orthant":
            return NonnegOrthant(int(d["dim"]))
    except (KeyError, TypeError) as exc:
        raise InputError(f"bad cone descriptor {d!r}: {exc}") from exc
    if kind in ("soc", "product"):
        raise ConfigurationError(f"cone type {kind!r} is not built on the device path")
    raise InputError(f"unknown cone type {kind!r}")
