"""The drop-in build without a GPU: the reference CLI linked with the B200
search must fail loudly (no CPU fallback) with the reference's error
convention (guarded(), tools/cli.cpp: exit 3 for non-spec errors), while the
reference CPU front end built from the same sources succeeds."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

from conftest import ROOT, gpu_available
from paper_2405_16256_b200 import configs

PLAN_B200 = os.path.join(ROOT, "integration", "_build", "hetplan_plan_b200")
PLAN_REF = os.path.join(ROOT, "oracle", "_ref", "hetplan_plan_ref")


def _inputs(d):
    docs = configs.config("C0", full=False)
    paths = []
    for k in ("model", "cluster", "train", "planner"):
        p = os.path.join(d, f"{k}.json")
        with open(p, "w") as f:
            json.dump(docs[k], f)
        paths += [f"--{k}", p]
    return paths


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU behaviour")
def test_dropin_cli_fails_loudly_without_gpu(tmp_path):
    if not os.path.exists(PLAN_B200):
        pytest.skip("integration not built (needs /root/reference at build time)")
    r = subprocess.run([PLAN_B200, *_inputs(str(tmp_path)), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 3, (r.returncode, r.stderr)
    assert "CUDA" in r.stderr or "cuda" in r.stderr.lower()
    assert not os.path.exists(tmp_path / "o" / "plan.json")


def test_reference_cli_front_end_runs(tmp_path):
    if not os.path.exists(PLAN_REF):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([PLAN_REF, *_inputs(str(tmp_path)), "--out", str(tmp_path / "o")],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    for f in ("plan.json", "report.json", "search_log.ndjson"):
        assert os.path.exists(tmp_path / "o" / f)
