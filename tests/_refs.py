"""Test-side independent references (brute force from the definitions) and golden parsing.

These are written from the definitions in SURVEY.md §8(c) / PAPER.md, independently of both
``oracle/`` and the CUDA path, and only for tiny inputs: O(N^2) loops in numpy.
"""
from __future__ import annotations

import itertools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def brute_edt_sq(labels: np.ndarray, border: bool) -> np.ndarray:
    """D(p) = min over sites |p-s|^2; sites = elements with another label (+ virtual border).

    Returns int64 array, 0 on background, -1 where no site exists.
    """
    lab = np.asarray(labels)
    shape = lab.shape
    coords = np.stack(np.meshgrid(*[np.arange(s) for s in shape], indexing="ij"), -1).reshape(-1, lab.ndim)
    flat = lab.reshape(-1)
    out = np.zeros(flat.size, np.int64)
    for i in np.nonzero(flat)[0]:
        p = coords[i]
        sites = coords[flat != flat[i]]
        best = np.inf
        if len(sites):
            best = float(((sites - p) ** 2).sum(1).min())
        if border:
            for a, n in enumerate(shape):
                best = min(best, (p[a] + 1) ** 2, (n - p[a]) ** 2)
        out[i] = -1 if best == np.inf else int(best)
    return out.reshape(shape)


def brute_lt_sq(labels: np.ndarray, D: np.ndarray) -> np.ndarray:
    """LT^2(p) = max{D(q): label(q)=label(p), |p-q|^2 < D(q)} by all-pairs search."""
    lab = np.asarray(labels)
    shape = lab.shape
    coords = np.stack(np.meshgrid(*[np.arange(s) for s in shape], indexing="ij"), -1).reshape(-1, lab.ndim)
    flat = lab.reshape(-1)
    Df = np.asarray(D).reshape(-1).astype(np.int64)
    out = np.zeros(flat.size, np.int64)
    for i in np.nonzero(flat)[0]:
        same = np.nonzero(flat == flat[i])[0]
        d2 = ((coords[same] - coords[i]) ** 2).sum(1)
        cov = d2 < Df[same]
        out[i] = Df[same][cov].max() if cov.any() else 0
    return out.reshape(shape)


def brute_shell(labels: np.ndarray, border: bool) -> np.ndarray:
    """Face-neighbour (4/6-conn) shell: some face neighbour has another label (or border)."""
    lab = np.asarray(labels)
    out = np.zeros(lab.shape, bool)
    for idx in itertools.product(*[range(s) for s in lab.shape]):
        if lab[idx] == 0:
            continue
        for a in range(lab.ndim):
            for s in (-1, 1):
                q = list(idx)
                q[a] += s
                if q[a] < 0 or q[a] >= lab.shape[a]:
                    out[idx] |= border
                elif lab[tuple(q)] != lab[idx]:
                    out[idx] = True
    return out


def load_spec_examples() -> dict:
    """Parse tests/golden/spec_examples.txt into {name: {key: value}}."""
    path = os.path.join(GOLDEN, "spec_examples.txt")
    cases, cur, key, rows = {}, None, None, []

    def flush():
        nonlocal key, rows
        if cur is not None and key is not None and rows:
            cases[cur][key] = np.array(rows, np.int64).reshape(cases[cur]["shape"])
        key, rows = None, []

    for raw in open(path):
        line = raw.split("#", 1)[0].strip() if raw.lstrip().startswith("#") else raw.strip()
        if not line:
            continue
        if line.startswith("["):
            flush()
            name = line[1:line.index("]")]
            meta = dict(kv.split("=") for kv in line[line.index("]") + 1:].split())
            cur = name
            cases[cur] = dict(ndim=int(meta["ndim"]), shape=tuple(int(v) for v in meta["shape"].split(",")))
            continue
        toks = line.split()
        if toks[0] in ("labels", "d2", "lt2", "shell"):
            flush()
            key = toks[0]
            continue
        if toks[0].lstrip("-").isdigit() and key is not None:
            rows.extend(int(t) for t in toks)
            continue
        flush()
        vals = [float(t) if "." in t else int(t) for t in toks[1:]]
        cases[cur][toks[0]] = vals[0] if len(vals) == 1 else vals
    flush()
    return cases


def load_closed_forms() -> dict:
    with open(os.path.join(GOLDEN, "closed_forms.json")) as f:
        return json.load(f)
