"""Profile calibration: measured transformer-layer timings -> per-group
compute_efficiency and bwd_fwd_ratio. Host-only and cold;
it runs once before a search, upstream of the per-group scalars the GPU
tables are built from.

    records, diags = parse_profiles(text)              profile.cpp:63-86
    cluster, diags = calibrate(records, model, cluster) profile.cpp:88-135
    docs, diags    = calibrate_docs(docs, text)         cli.cpp:107-114

Same arithmetic in the same order as the reference (IEEE doubles, no
contraction): efficiency = (layer_flops / (tp * peak * 1e12)) / (fwd_ms / 1e3)
per record, median per group, clamped to 1.5; ratio = median(bwd/fwd), raised
to 1.0. Diagnostic strings follow the reference; for a line that is not
valid JSON the text after "line N: " is this parser's, not nlohmann's.
"""
from __future__ import annotations

import copy
import json
from dataclasses import dataclass
from typing import Dict, List, Tuple

from .abi import ConfigError

EFFICIENCY_CLAMP = 1.5  # profile.cpp:32
OP_KINDS = ("transformer_layer", "embedding", "lm_head")


@dataclass
class ProfileRecord:
    """profile.hpp:29-40"""
    device_type: str
    op_kind: str = "transformer_layer"
    micro_batch: int = 1
    seq_length: int = 0
    hidden: int = 0
    tp_degree: int = 1
    fwd_ms: float = 0.0
    bwd_ms: float = 0.0


_TYPE_NAMES = {type(None): "null", bool: "boolean", int: "number", float: "number", str: "string",
               list: "array", dict: "object"}


def _tname(v) -> str:
    return _TYPE_NAMES.get(type(v), "unknown")


class _RecordError(Exception):
    pass


def _int(v) -> int:
    # nlohmann get<integer>: numbers and booleans convert (floats truncate)
    if isinstance(v, (bool, int)):
        return int(v)
    if isinstance(v, float):
        return int(v)
    raise _RecordError(f"[json.exception.type_error.302] type must be number, but is {_tname(v)}")


def _float(v) -> float:
    if isinstance(v, (bool, int, float)):
        return float(v)
    raise _RecordError(f"[json.exception.type_error.302] type must be number, but is {_tname(v)}")


def _str(v) -> str:
    if isinstance(v, str):
        return v
    raise _RecordError(f"[json.exception.type_error.302] type must be string, but is {_tname(v)}")


def _record_from_json(j) -> ProfileRecord:
    """record_from_json, profile.cpp:41-56 (field order = check order)."""
    def at(k):
        if not isinstance(j, dict):
            raise _RecordError(f"[json.exception.type_error.304] cannot use at() with {_tname(j)}")
        if k not in j:
            raise _RecordError(f"[json.exception.out_of_range.403] key '{k}' not found")
        return j[k]

    def value(k, default):
        if not isinstance(j, dict):
            raise _RecordError(f"[json.exception.type_error.306] cannot use value() with {_tname(j)}")
        return j[k] if k in j else default

    r = ProfileRecord(device_type=_str(at("device_type")))
    op = _str(value("op_kind", "transformer_layer"))
    if op not in OP_KINDS:
        raise _RecordError(f"unknown op_kind '{op}'")
    r.op_kind = op
    r.micro_batch = _int(at("micro_batch"))
    r.seq_length = _int(at("seq_length"))
    r.hidden = _int(at("hidden"))
    r.tp_degree = _int(value("tp_degree", 1))
    r.fwd_ms = _float(at("fwd_ms"))
    r.bwd_ms = _float(at("bwd_ms"))
    if r.fwd_ms <= 0 or r.bwd_ms <= 0:
        raise _RecordError("fwd_ms and bwd_ms must be > 0")
    if r.micro_batch < 1 or r.seq_length < 1 or r.hidden < 1:
        raise _RecordError("micro_batch, seq_length, hidden must be >= 1")
    if r.tp_degree < 1:
        raise _RecordError("tp_degree must be >= 1")
    return r


def _no_constants(name):
    raise ValueError(f"invalid literal {name}")


def parse_profiles(text: str) -> Tuple[List[ProfileRecord], List[str]]:
    """parse_profiles, profile.cpp:63-86: one JSON record per line; blank
    lines skipped; bad lines become diagnostics "line N: ..."."""
    records, diags = [], []
    for n, line in enumerate(text.split("\n"), start=1):
        if line.strip(" \t\r") == "":
            continue
        try:
            j = json.loads(line, parse_constant=_no_constants)
        except ValueError as e:
            diags.append(f"line {n}: [json.exception.parse_error.101] parse error: {e}")
            continue
        try:
            records.append(_record_from_json(j))
        except _RecordError as e:
            diags.append(f"line {n}: {e}")
    return records, diags


def _median(v: List[float]) -> float:
    v = sorted(v)
    n = len(v)
    return v[n // 2] if n % 2 == 1 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def _layer_flops_fwd(B: int, L: int, H: int) -> float:
    """layer_flops (cost_model.cpp:29-35), forward."""
    Bd, Ld, Hd = float(B), float(L), float(H)
    return 24.0 * Bd * Ld * Hd * Hd + 4.0 * Bd * Ld * Ld * Hd


def calibrate(records: List[ProfileRecord], model: Dict, cluster: Dict) -> Tuple[Dict, List[str]]:
    """calibrate, profile.cpp:88-135, on the reference's JSON documents.
    Returns the calibrated cluster document and the diagnostics."""
    out = copy.deepcopy(cluster)
    groups = out.get("groups", [])
    by_name = {}
    for g in groups:
        by_name.setdefault(g["name"], g)  # find_group: first match
    diags: List[str] = []
    eff: Dict[str, List[float]] = {}
    ratio: Dict[str, List[float]] = {}
    for r in records:
        g = by_name.get(r.device_type)
        if g is None:
            diags.append(f"record for unknown device_type '{r.device_type}' skipped")
            continue
        if r.op_kind != "transformer_layer":
            continue
        flops = _layer_flops_fwd(r.micro_batch, r.seq_length, r.hidden)
        ideal_s = flops / (r.tp_degree * float(g["peak_tflops"]) * 1e12)
        eff.setdefault(r.device_type, []).append(ideal_s / (r.fwd_ms / 1e3))
        ratio.setdefault(r.device_type, []).append(r.bwd_ms / r.fwd_ms)
    for g in groups:
        name = g["name"]
        if name not in eff:
            continue
        e = _median(eff[name])
        if e > EFFICIENCY_CLAMP:
            diags.append(f"group '{name}': calibrated efficiency {e:f} clamped to 1.5 "
                         "(peak_tflops entry looks wrong)")
            e = EFFICIENCY_CLAMP
        g["compute_efficiency"] = e
        q = _median(ratio[name])
        if q < 1.0:
            diags.append(f"group '{name}': profiled bwd/fwd ratio {q:f} raised to 1.0")
            q = 1.0
        g["bwd_fwd_ratio"] = q
    return out, diags


def calibrate_docs(docs: Dict[str, dict], profiles_text: str) -> Tuple[Dict[str, dict], List[str]]:
    """What `hetplan plan --profiles F` does before searching (cli.cpp:107-114):
    parse, calibrate the cluster, return new documents plus the diagnostics
    ("profiles: ..." then "calibration: ...")."""
    if "model" not in docs or "cluster" not in docs:
        raise ConfigError("calibrate_docs needs the model and cluster documents")
    records, pd = parse_profiles(profiles_text)
    cluster, cd = calibrate(records, docs["model"], docs["cluster"])
    out = dict(docs)
    out["cluster"] = cluster
    return out, [f"profiles: {d}" for d in pd] + [f"calibration: {d}" for d in cd]
