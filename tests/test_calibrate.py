"""Profile calibration (profile.cpp:63-135) against the
compiled reference: calibrated per-group scalars bit for bit and the
diagnostics list, on seeded random profile sets with unknown device types,
clamped efficiencies, raised ratios, invalid records and blank lines."""
from __future__ import annotations

import json
import random
import struct

import pytest

from oracle import ref
from paper_2405_16256_b200 import calibrate, configs

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def bits(x: float) -> str:
    return "%016x" % struct.unpack("<Q", struct.pack("<d", x))[0]


def random_profiles(rng: random.Random, groups) -> str:
    lines = []
    for _ in range(rng.randrange(0, 14)):
        kind = rng.random()
        g = rng.choice(groups + ["ghost"]) if rng.random() < 0.9 else "ghost"
        rec = {"device_type": g, "micro_batch": rng.choice([1, 2, 4]), "seq_length": rng.choice([1024, 2048, 4096]),
               "hidden": rng.choice([4096, 8192]), "tp_degree": rng.choice([1, 2, 4, 8]),
               "fwd_ms": round(rng.uniform(0.05, 40.0), 3), "bwd_ms": round(rng.uniform(0.05, 90.0), 3)}
        if rng.random() < 0.3:
            rec["op_kind"] = rng.choice(["transformer_layer", "embedding", "lm_head"])
        if kind < 0.05:
            rec["op_kind"] = "attention"
        elif kind < 0.10:
            rec["fwd_ms"] = 0
        elif kind < 0.14:
            del rec["hidden"]
        elif kind < 0.17:
            rec["tp_degree"] = 0
        elif kind < 0.20:
            rec["micro_batch"] = "two"
        elif kind < 0.23:
            rec["fwd_ms"] = 1e-4  # efficiency far above 1.5 -> clamp
        line = json.dumps(rec)
        if rng.random() < 0.1:
            lines.append("   ")
        lines.append(line)
    return "\n".join(lines) + ("\n" if rng.random() < 0.5 else "")


def test_calibrate_matches_reference():
    rng = random.Random(5)
    for k in range(200):
        docs = configs.config(rng.choice(["C0", "C1", "C2", "C4:nvidia+amd"]), full=False)
        groups = [g["name"] for g in docs["cluster"]["groups"]]
        text = random_profiles(rng, groups)
        want = ref.calibrate(docs["model"], docs["cluster"], text)
        assert want["status"] == 0, want
        got_docs, diags = calibrate.calibrate_docs(docs, text)
        assert diags == want["diagnostics"], (k, text)
        for g, w in zip(got_docs["cluster"]["groups"], want["groups"]):
            assert g["name"] == w["name"]
            assert bits(float(g.get("compute_efficiency", 1.0))) == w["compute_efficiency_bits"], (k, g["name"])
            assert bits(float(g.get("bwd_fwd_ratio", 2.0))) == w["bwd_fwd_ratio_bits"], (k, g["name"])


def test_calibration_known_answer():
    """Hand-checked record: 24*1*4096*8192^2 + 4*1*4096^2*8192 = 7.146825580544e12
    forward FLOPs; at tp 8 x 383 TFLOP/s the ideal time is 2.3325e-3 s, so
    fwd_ms 9.52 gives efficiency 0.24501... and bwd/fwd 2.0001."""
    docs = configs.config("C0", full=False)
    text = json.dumps({"device_type": "amd", "micro_batch": 1, "seq_length": 4096, "hidden": 8192,
                       "tp_degree": 8, "fwd_ms": 9.52, "bwd_ms": 19.041})
    out, diags = calibrate.calibrate_docs(docs, text)
    amd = [g for g in out["cluster"]["groups"] if g["name"] == "amd"][0]
    flops = 24.0 * 4096 * 8192 * 8192 + 4.0 * 4096 * 4096 * 8192
    assert amd["compute_efficiency"] == (flops / (8 * 383.0 * 1e12)) / (9.52 / 1e3)
    assert abs(amd["compute_efficiency"] - 0.2450) < 1e-3
    assert amd["bwd_fwd_ratio"] == 19.041 / 9.52
    assert diags == []
    want = ref.calibrate(docs["model"], docs["cluster"], text)
    assert bits(amd["compute_efficiency"]) == want["groups"][[g["name"] for g in want["groups"]].index("amd")][
        "compute_efficiency_bits"]
