"""Bundled instances (the reference's datasets.py:15-40 API).

The reference ships chr12a, esc32e (QAPLIB reconstructions with their .sln
files) and two synthetic dense instances, rand26 and rand150, as text files
(pkg/src/qapswarm/data/README.md gives their provenance).  Here they are
packed as arrays in ``data/bundled.npz`` (scripts/make_bundled.py);
:func:`data_path` writes the QAPLIB-format text of a file on first use, so
code that opens the path keeps working.
"""

from __future__ import annotations

import os
import tempfile
from functools import lru_cache
from pathlib import Path

import numpy as np

from .instance import (QapInstance, ReferenceSolution, format_instance,
                       format_reference_solution, load_instance, load_reference_solution)

_NPZ = Path(__file__).resolve().parent / "data" / "bundled.npz"

# published reference values of the bundled benchmark instances (datasets.py:15-18)
KNOWN_BEST = {"chr12a": 9552, "esc32e": 2}


@lru_cache(maxsize=1)
def _arrays() -> dict:
    with np.load(_NPZ) as z:
        return {k: z[k] for k in z.files}


def _names() -> list[str]:
    return sorted({k.split("__")[0] for k in _arrays()})


@lru_cache(maxsize=1)
def _text_dir() -> Path:
    d = Path(tempfile.gettempdir()) / f"qsb_bundled_{os.getuid()}_{_NPZ.stat().st_mtime_ns}"
    d.mkdir(parents=True, exist_ok=True)
    return d


def _instance_from_arrays(name: str) -> QapInstance:
    a = _arrays()
    return QapInstance(name, int(a[f"{name}__flow"].shape[0]), a[f"{name}__flow"],
                       a[f"{name}__distance"])


def data_path(name: str) -> Path:
    """Filesystem path of a bundled file, e.g. ``chr12a.dat`` or
    ``chr12a.sln``; FileNotFoundError for unknown names."""
    stem, dot, ext = name.rpartition(".")
    a = _arrays()
    if not dot or stem not in _names() or ext not in ("dat", "sln") or \
            (ext == "sln" and f"{stem}__sln_perm" not in a):
        raise FileNotFoundError(f"no bundled data file named {name!r}")
    p = _text_dir() / name
    if not p.is_file():
        if ext == "dat":
            text = format_instance(_instance_from_arrays(stem))
        else:
            cost = a[f"{stem}__sln_cost"].item()
            text = format_reference_solution(
                ReferenceSolution(int(a[f"{stem}__sln_perm"].size), cost, a[f"{stem}__sln_perm"]))
        tmp = p.with_suffix(p.suffix + f".{os.getpid()}")
        tmp.write_text(text)
        tmp.replace(p)
    return p


def list_bundled() -> list[str]:
    """File names of the bundled instances (``*.dat``)."""
    return [f"{n}.dat" for n in _names()]


def load_bundled(name: str) -> QapInstance:
    """A bundled instance by stem, with its published value as ``known_best``."""
    return load_instance(data_path(f"{name}.dat"), known_best=KNOWN_BEST.get(name))


def load_bundled_solution(name: str) -> ReferenceSolution:
    return load_reference_solution(data_path(f"{name}.sln"))
