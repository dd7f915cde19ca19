"""Parser for the hand-worked fixtures in tests/golden/*.txt (letters -> packed labels)."""
from __future__ import annotations

import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EMPTY = 0xFFFFFFFF


def _pack(x: int, y: int) -> int:
    # The fixture files define a label as (y << 16) | x in their header comments.
    return (y << 16) | x


def load(name: str) -> dict:
    path = os.path.join(GOLDEN_DIR, name)
    out = {"seeds": {}, "prev_seeds": {}, "disp": {}, "grids": {}}
    lines = [ln.rstrip("\n") for ln in open(path, encoding="utf-8")]
    lines = [ln for ln in lines if ln.strip() and not ln.lstrip().startswith("#")]
    i = 0
    while i < len(lines):
        tok = lines[i].split()
        if tok[0] == "N":
            out["N"] = int(tok[1])
        elif tok[0] == "seed":
            out["seeds"][tok[1]] = (int(tok[2]), int(tok[3]))
        elif tok[0] == "prev_seed":
            out["prev_seeds"][tok[1]] = (int(tok[2]), int(tok[3]))
        elif tok[0] == "disp":
            out["disp"][tok[1]] = (int(tok[2]), int(tok[3]))
        elif tok[0] == "d_max":
            out["d_max"] = int(tok[1])
        elif tok[0] == "schedule":
            out["schedule"] = [int(t) for t in tok[1:]]
        elif tok[0] == "grid":
            N = out["N"]
            rows = [lines[i + 1 + r].split() for r in range(N)]
            out["grids"][tok[1]] = rows
            i += N
        i += 1
    return out


def grid(fx: dict, name: str) -> np.ndarray:
    """Grid `name` as (N, N) uint32 labels; 'prev' uses the prev_seed letters."""
    table = fx["prev_seeds"] if name == "prev" else fx["seeds"]
    rows = fx["grids"][name]
    N = fx["N"]
    g = np.empty((N, N), dtype=np.uint32)
    for y in range(N):
        for x in range(N):
            t = rows[y][x]
            g[y, x] = EMPTY if t == "." else _pack(*table[t])
    return g


def seeds_xy(fx: dict, key: str = "seeds") -> np.ndarray:
    pts = [fx[key][k] for k in sorted(fx[key])]
    return np.array([c for p in pts for c in p], dtype=np.uint16)


def disp_xy(fx: dict) -> np.ndarray:
    pts = [fx["disp"][k] for k in sorted(fx["disp"])]
    return np.array([c for p in pts for c in p], dtype=np.int16)


def load_seed_runs(name: str) -> dict:
    """Fixtures written as `seeds old_x old_y disp_x disp_y count` runs (index order) plus
    `expect px py lx ly` lines (pixel (px,py) ends with the label of (lx,ly))."""
    out = {"old": [], "disp": [], "expect": []}
    for ln in open(os.path.join(GOLDEN_DIR, name), encoding="utf-8"):
        tok = ln.split("#", 1)[0].split()
        if not tok:
            continue
        if tok[0] in ("N", "d_max"):
            out[tok[0]] = int(tok[1])
        elif tok[0] == "schedule":
            out["schedule"] = [int(t) for t in tok[1:]]
        elif tok[0] == "seeds":
            ox, oy, dx, dy, cnt = (int(t) for t in tok[1:])
            out["old"] += [(ox, oy)] * cnt
            out["disp"] += [(dx, dy)] * cnt
        elif tok[0] == "expect":
            px, py, lx, ly = (int(t) for t in tok[1:])
            out["expect"].append((px, py, _pack(lx, ly)))
    out["old_xy"] = np.array([c for p in out["old"] for c in p], dtype=np.uint16)
    out["disp_xy"] = np.array([c for p in out["disp"] for c in p], dtype=np.int16)
    return out
