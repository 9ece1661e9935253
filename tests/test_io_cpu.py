"""Run artefacts (q/io.py) are byte-compatible with the reference's: the
trajectory JSONL and the metrics CSV written from the same data equal the
files the reference wrote (tests/golden/trajectory.jsonl, metrics.csv)."""

import csv
import os

import numpy as np
import torch

from golden_utils import GOLDEN, load


def test_trajectory_jsonl_matches_reference(tmp_path):
    from paper_2509_10247_b200 import io as qio

    z = load("io_inputs")
    out = str(tmp_path / "t.jsonl")
    tw = qio.TrajectoryWriter(out, env_limit=2)
    for step in range(2):
        t = lambda k: torch.as_tensor(z[f"t{step}_{k}"])  # noqa: E731  (device arrays in practice)
        tw.write_step(step, {"p": t("p"), "v": t("v")}, t("a"), t("rc"), t("rg"), t("term"), t("trunc"))
    tw.close()
    ref = os.path.join(GOLDEN, "trajectory.jsonl")
    assert open(out).read() == open(ref).read()
    recs = qio.read_trajectory(out)
    assert len(recs) == 4 and recs[3]["env"] == 1 and recs[3]["step"] == 1 and recs[1]["truncated"] is True


def test_metrics_csv_matches_reference(tmp_path):
    from paper_2509_10247_b200 import io as qio

    ref = os.path.join(GOLDEN, "metrics.csv")
    rows = list(csv.DictReader(open(ref)))
    out = str(tmp_path / "m.csv")
    mw = qio.MetricsWriter(out)
    for r in rows:
        mw.write({"update": int(r["update"]), "loss": float(r["loss"]), "steps_per_sec": float(r["steps_per_sec"])})
    mw.close()
    assert mw.rows == 3
    assert open(out).read() == open(ref).read()
