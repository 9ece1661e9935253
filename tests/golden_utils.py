"""Fixture loading shared by the CPU (oracle) and GPU (parity) tests."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import quadsim_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def scene_from_json(text) -> O.Scene:
    """Scene JSON v1 (q/world.py:72-111) -> oracle Scene."""
    d = json.loads(str(text))
    prims = {
        "spheres": np.array(d["spheres"], dtype=np.float64).reshape(-1, 4),
        "boxes": np.array(d["boxes"], dtype=np.float64).reshape(-1, 6),
        "cylinders": np.array(d["cylinders"], dtype=np.float64).reshape(-1, 5),
        "ground_z": d["ground_z"],
    }
    gates = [(np.array(g["center"]), np.array(g["normal"]), g["inner_radius"], g["frame_width"])
             for g in d["gates"]]
    return O.Scene(prims=prims, bounds_lo=np.array(d["bounds_lo"]), bounds_hi=np.array(d["bounds_hi"]),
                   spawn=np.array(d["spawn"]), goal=np.array(d["goal"]), gates=gates, seed=d["seed"],
                   style=d["style"])


# the TaskConfig keyword sets of tests/golden/make_golden.py:TASK_CASES, restated
# without importing the reference (which does not exist on the GPU box)
TASK_CASES = {
    "pos_pmc": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=64, episode_len=10)),
    "pos_pmd": dict(cfg=dict(task="position", dynamics="pm_discrete", n_envs=64, episode_len=10)),
    "pos_full": dict(cfg=dict(task="position", dynamics="full", n_envs=32, episode_len=7)),
    "pos_pmc_dr": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=16, episode_len=6),
                       randomization=dict(action_scale=(0.7, 1.0))),
    "pos_form": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=8, n_agents=3,
                              episode_len=9, formation="line")),
    "avoid_depth": dict(cfg=dict(task="avoidance", dynamics="pm_continuous", n_envs=6, episode_len=8,
                                 sensor="depth", density=0.12)),
    "avoid_lidar_indoor": dict(cfg=dict(task="avoidance", dynamics="full", n_envs=4, episode_len=6,
                                        sensor="lidar", style="indoor", density=0.12),
                               lidar=(24, 3)),
    "avoid_form": dict(cfg=dict(task="avoidance", dynamics="pm_discrete", n_envs=4, n_agents=2,
                                episode_len=7, density=0.1, formation="line", formation_side=1.5)),
    "racing": dict(cfg=dict(task="racing", dynamics="pm_continuous", n_envs=8, episode_len=30,
                            n_gates=3, gate_spread=6.0)),
    "pos_events": dict(cfg=dict(task="position", dynamics="pm_continuous", n_envs=24, episode_len=20)),
    "pos_full_events": dict(cfg=dict(task="position", dynamics="full", n_envs=16, episode_len=20)),
    "avoid_collide": dict(cfg=dict(task="avoidance", dynamics="pm_continuous", n_envs=6, episode_len=20,
                                   density=0.2)),
    "pos_simp": dict(cfg=dict(task="position", dynamics="simplified", n_envs=24, episode_len=7)),
}

STATE_KEYS = {"full": ("p", "v", "q", "w"), "pm_continuous": ("p", "v", "a_lat"),
              "pm_discrete": ("p", "v", "u_prev"), "simplified": ("p", "v", "R")}


def oracle_config(name) -> O.Config:
    spec = TASK_CASES[name]
    cfg = O.Config(**spec["cfg"])
    if "randomization" in spec:
        cfg.randomization = O.RandomizationSpec(**spec["randomization"])
    if "lidar" in spec:
        n_az, n_el = spec["lidar"]
        cfg.lidar = (n_az, n_el, 2 * np.pi, np.deg2rad(30.0), 20.0)
    return cfg


def fixture_state(z, t, model):
    return {k: z[f"s{t}_{k}"] for k in STATE_KEYS[model]}
