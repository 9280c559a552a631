"""Write the committed MoA rule tables ``moa_workloads/rules/<C>.json``.

Synthetic MoA configurations (SURVEY.md §8(d) "synthetic MoA span
generator"): rules (alpha, beta) from the paper's 6 x 9 grid,
at most two distinct rules per layer, and a
per-layer density profile shaped like PAPER.md:1229-1230 / 1264 ("masks in
the initial and middle layers exhibit high density ... in the final layers,
most heads require low density, while few need high density").  GQA configs
assign one rule per kv-group (reading c10).  The overall mean density
(reading c11) is tuned to the config's target within 1%.

Only ``oracle/`` is used for span/window/density arithmetic, so the tables are
inputs that never came from the CUDA path.  Run:

    python tools/make_rule_tables.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import density, span_of, window_of  # noqa: E402
from moa_workloads.configs import ALPHA_GRID, BETA_GRID, CONFIGS  # noqa: E402

RULES = [(a, b) for a in ALPHA_GRID for b in BETA_GRID]


def profile(x: float) -> float:
    """Relative density vs normalised depth x in [0, 1]: dense first layers,
    a medium plateau with a second bump, sparse last layers (two local
    minima)."""
    pts = [(0.0, 1.0), (0.12, 1.0), (0.35, 0.55), (0.5, 0.7), (0.65, 0.45),
           (0.8, 0.3), (1.0, 0.3)]
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        if x <= x1:
            return y0 + (y1 - y0) * (x - x0) / (x1 - x0)
    return pts[-1][1]


def rule_density(rule, N, s):
    return density([window_of(span_of(rule[0], rule[1], N), s)], s, N)


def best_layer(target, H, N, s, dens, late):
    best = None
    max_out = max(1, H // 4)
    for i, ri in enumerate(RULES):
        for j, rj in enumerate(RULES):
            if i == j:
                continue
            if late and dens[j] <= dens[i]:
                continue           # late layers: the outliers are the dense heads
            for n_out in range(1, max_out + 1):
                dl = ((H - n_out) * dens[i] + n_out * dens[j]) / H
                err = abs(dl - target)
                key = (round(err, 6), -n_out if late else n_out)
                if best is None or key < best[0]:
                    best = (key, i, j, n_out, dl)
    return best


def build(cfg, seed):
    N, s = cfg.N, cfg.n_sink
    H = cfg.hkv if cfg.group > 1 else cfg.hq       # rule units
    L = cfg.layers
    dens = [rule_density(r, N, s) for r in RULES]
    rng = np.random.default_rng(seed)
    perms = [rng.permutation(H) for _ in range(L)]

    def realise(c):
        layers = []
        for l in range(L):
            x = l / max(1, L - 1)
            t = min(1.0, max(s / N, c * profile(x)))
            _, i, j, n_out, dl = best_layer(t, H, N, s, dens, late=x >= 0.5)
            layers.append((i, j, n_out, dl))
        mean = float(np.mean([dl for *_, dl in layers]))
        return layers, mean

    lo, hi = 0.0, 4.0
    layers, mean = realise(1.0)
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        layers, mean = realise(mid)
        if abs(mean - cfg.target_density) < 0.002:
            break
        if mean < cfg.target_density:
            lo = mid
        else:
            hi = mid
    alpha = np.zeros((L, cfg.hq))
    beta = np.zeros((L, cfg.hq))
    for l, (i, j, n_out, _) in enumerate(layers):
        unit_rule = [i] * H
        for u in perms[l][:n_out]:
            unit_rule[u] = j
        for h in range(cfg.hq):
            r = RULES[unit_rule[h // cfg.group]]
            alpha[l, h], beta[l, h] = r
    windows = [[window_of(span_of(alpha[l, h], beta[l, h], N), s) for h in range(cfg.hq)]
               for l in range(L)]
    achieved = float(np.mean([density(w, s, N) for w in windows]))
    return {
        "config": cfg.name, "N": N, "n_sink": s, "layers": L, "hq": cfg.hq,
        "hkv": cfg.hkv, "seed": seed, "target_density": cfg.target_density,
        "achieved_density_oracle": achieved,
        "generator": "tools/make_rule_tables.py (oracle.span_of/window_of/density)",
        "alpha": alpha.tolist(), "beta": beta.tolist(),
    }


def main():
    out_dir = os.path.join(ROOT, "moa_workloads", "rules")
    os.makedirs(out_dir, exist_ok=True)
    for name, cfg in CONFIGS.items():
        if cfg.target_density is None:
            continue
        t = build(cfg, seed=cfg.seed_base)
        with open(os.path.join(out_dir, f"{name}.json"), "w") as f:
            json.dump(t, f)
        print(name, "density", round(t["achieved_density_oracle"], 4),
              "target", cfg.target_density)


if __name__ == "__main__":
    main()
