"""Approximant data type and its JSON format (rbainv.rba, rba.py:42-136,474-500).

The common-pole fit itself (rba.py:280-378) is offline and out of scope: the
frozen approximants of the BASELINE configs (fitted with the reference's
``fit_common_pole``) ship as JSON in ``data/`` and load into this type; a
reference ``RationalApproximant`` is accepted everywhere duck-typed.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

__all__ = ["TimeChannels", "RationalApproximant", "load_approximant", "save_approximant",
           "config_approximant"]

DATA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


@dataclass(frozen=True)
class TimeChannels:
    times: np.ndarray

    def __post_init__(self):
        t = np.atleast_1d(np.asarray(self.times, dtype=float))
        if t.size and (np.any(t <= 0) or np.any(np.diff(t) <= 0)):
            raise ValueError("times must be strictly increasing and positive")
        object.__setattr__(self, "times", t)

    @property
    def count(self) -> int:
        return self.times.size

    @classmethod
    def logspaced(cls, t_min, t_max, count):
        return cls(np.geomspace(t_min, t_max, count))


@dataclass(frozen=True)
class RationalApproximant:
    poles: np.ndarray
    residues: np.ndarray
    spectral_interval: tuple
    fit_error: float
    channels: TimeChannels
    converged: bool = True
    iterations: int = 0

    def __post_init__(self):
        poles = np.atleast_1d(np.asarray(self.poles, dtype=complex))
        residues = np.asarray(self.residues, dtype=complex).reshape(poles.size, -1)
        if np.any(poles.imag <= 0):
            raise ValueError("poles must lie strictly in the upper half-plane")
        object.__setattr__(self, "poles", poles)
        object.__setattr__(self, "residues", residues)

    @property
    def pole_count(self) -> int:
        return self.poles.size

    def eval(self, x) -> np.ndarray:
        x = np.atleast_1d(np.asarray(x, dtype=float))
        r = 1.0 / (x[:, None] - self.poles[None, :])
        return 2.0 * np.real(r @ self.residues)


def save_approximant(approx, path) -> None:
    """Same layout as rba.py:474-485."""
    doc = {
        "times": approx.channels.times.tolist(),
        "poles": [[p.real, p.imag] for p in approx.poles],
        "residues": [[[a.real, a.imag] for a in approx.residues[:, j]]
                     for j in range(approx.channels.count)],
        "interval": list(approx.spectral_interval),
        "fit_error": approx.fit_error,
    }
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_approximant(path) -> RationalApproximant:
    """rba.py:488-500"""
    with open(path) as fh:
        doc = json.load(fh)
    poles = np.array([complex(re, im) for re, im in doc["poles"]])
    res = np.array([[complex(re, im) for re, im in chan] for chan in doc["residues"]])
    return RationalApproximant(poles=poles, residues=res.T,
                               spectral_interval=tuple(doc["interval"]),
                               fit_error=float(doc["fit_error"]),
                               channels=TimeChannels(np.array(doc["times"])))


def config_approximant(name: str) -> RationalApproximant:
    """Frozen approximant of a BASELINE config (C1: 8 poles; C2-C4: 16; C5: 20),
    each fitted by the reference's ``fit_common_pole`` on its own config's
    spectral interval (tests/golden/make_golden.py: C2 without air reaches
    8.4e10; C1, C3, C4, C5 with 1e-8 S/m air reach ~8e15)."""
    key = name.upper()
    if key not in ("C1", "C2", "C3", "C4", "C5"):
        raise ValueError(f"unknown config {name}")
    return load_approximant(os.path.join(DATA_DIR, f"approx_{key}.json"))
