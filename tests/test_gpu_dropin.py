"""The drop-in boundary end to end: the reference's own code
with hetplan::search (planner.hpp:115-116) replaced by
integration/hetplan_search_b200.cpp, running on the GPU.

* integration/_build/libhetplan_dropin.so — the unmodified reference library
  plus the B200 search, driven through the same JSON driver as oracle/_ref:
  plans, iteration-time bits, candidate counts and search logs equal the
  golden fixtures of the reference.
* integration/_build/hetplan_plan_b200 — the reference CLI's `plan` command
  (tools/cli.cpp:216-260) over the B200 search: plan.json, report.json,
  search_log.ndjson, stdout and exit codes byte-identical to the same front
  end over the reference CPU search (oracle/_ref/hetplan_plan_ref).
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import random
import subprocess

import pytest

from conftest import ROOT, load_golden
from instances import random_instance
from paper_2405_16256_b200 import configs

pytestmark = pytest.mark.gpu

DROPIN = os.path.join(ROOT, "integration", "_build", "libhetplan_dropin.so")
PLAN_B200 = os.path.join(ROOT, "integration", "_build", "hetplan_plan_b200")
PLAN_REF = os.path.join(ROOT, "oracle", "_ref", "hetplan_plan_ref")


def _need(path):
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build with `make -C integration` / `make -C oracle ref`")


@pytest.fixture(scope="module")
def dropin():
    _need(DROPIN)
    l = ctypes.CDLL(DROPIN)
    cp = ctypes.c_char_p
    l.ref_search_json.argtypes = [cp, cp, cp, cp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    l.ref_search_json.restype = ctypes.c_int
    l.ref_free.argtypes = [ctypes.c_void_p]

    def search(docs, want_log=False):
        out = ctypes.c_void_p()
        enc = [json.dumps(docs[k]).encode() for k in ("model", "cluster", "train", "planner")]
        l.ref_search_json(*enc, 1, int(want_log), ctypes.byref(out))
        s = ctypes.string_at(out.value).decode()
        l.ref_free(out)
        return json.loads(s)

    return search


def _digest(log):
    h = hashlib.sha256()
    for e in log:
        h.update(f"{e['candidate']}\t{e['time_bits']}\t{e['reason']}\n".encode())
    return h.hexdigest()


def test_dropin_library_matches_reference(dropin, search_cases):
    logs = {c["name"]: c for c in load_golden("search_logs.json")}
    for case in search_cases:
        r = dropin(case["docs"], want_log=True)
        assert r["status"] == case["status"], case["name"]
        if case["status"] != 0:
            assert r.get("reasons", []) == logs[case["name"]]["reasons"], case["name"]
            continue
        assert r["eval"]["iteration_bits"] == case["iteration_bits"], case["name"]
        assert r["plan"] == case["plan"], case["name"]
        assert (r["candidates_simulated"], r["candidates_pruned"]) == (
            case["candidates_simulated"], case["candidates_pruned"]), case["name"]
        assert len(r["log"]) == logs[case["name"]]["n"], case["name"]
        assert _digest(r["log"]) == logs[case["name"]]["sha256"], case["name"]


def test_dropin_winner_evaluation_matches_reference(dropin, search_cases):
    """SearchOutcome.eval (planner.cpp:681-684) comes from the B200 engine
    (hp_evaluate_plan_full), equal to the reference's PlanEvaluation: stage
    costs, compute ends, peak in-flight / memory, pipeline time, bubbles."""
    from oracle import ref
    n = 0
    for case in search_cases:
        if case["status"] != 0:
            continue
        got = dropin(case["docs"])["eval"]
        want = ref.search(case["docs"])["eval"]
        assert got == want, case["name"]
        n += 1
        if n >= 60:
            break


def _write_inputs(d, docs):
    paths = {}
    for k in ("model", "cluster", "train", "planner"):
        p = os.path.join(d, f"{k}.json")
        with open(p, "w") as f:
            json.dump(docs[k], f, indent=2)
        paths[k] = p
    return paths


def _run_plan(binary, paths, out):
    cmd = [binary, "--model", paths["model"], "--cluster", paths["cluster"], "--train", paths["train"],
           "--planner", paths["planner"], "--out", out, "--jobs", "4"]
    if "profiles" in paths:
        cmd += ["--profiles", paths["profiles"]]
    # NCCL_DEBUG asks NCCL (the drop-in's multi-GPU path, --jobs > 1) to print
    # its own diagnostics on stderr; compare the planners' output without it
    env = {k: v for k, v in os.environ.items() if k != "NCCL_DEBUG"}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    files = {}
    for name in ("plan.json", "report.json", "search_log.ndjson"):
        fp = os.path.join(out, name)
        if os.path.exists(fp):
            files[name] = open(fp, "rb").read()
    return r.returncode, r.stdout.replace(out, "<OUT>"), r.stderr, files


def _cli_cases():
    cases = [("C0-full", configs.config("C0", full=True)), ("C0-default", configs.config("C0", full=False)),
             ("C1-default", configs.config("C1", full=False)), ("C2u-full", configs.config("C2u", full=True))]
    rng = random.Random(7)
    for k in range(12):
        cases.append((f"rand{k}", random_instance(rng, k)))
    return cases


@pytest.mark.parametrize("name,docs", _cli_cases(), ids=lambda x: x if isinstance(x, str) else "")
def test_cli_plan_outputs_byte_identical(tmp_path, name, docs):
    _need(PLAN_B200)
    _need(PLAN_REF)
    paths = _write_inputs(str(tmp_path), docs)
    got = _run_plan(PLAN_B200, paths, str(tmp_path / "b200"))
    want = _run_plan(PLAN_REF, paths, str(tmp_path / "ref"))
    assert got[0] == want[0], (name, got[2], want[2])
    assert got[1].replace("/b200", "/X") == want[1].replace("/ref", "/X"), name
    assert got[2] == want[2], name
    assert sorted(got[3]) == sorted(want[3]), name
    for k in want[3]:
        assert got[3][k] == want[3][k], (name, k)


def _profiles(rng, groups):
    lines = []
    for g in groups:
        for _ in range(rng.randrange(1, 4)):
            lines.append(json.dumps({"device_type": g, "micro_batch": rng.choice([1, 2]), "seq_length": 4096,
                                     "hidden": 8192, "tp_degree": rng.choice([4, 8]),
                                     "fwd_ms": round(rng.uniform(5.0, 30.0), 3),
                                     "bwd_ms": round(rng.uniform(10.0, 70.0), 3)}))
    lines.append(json.dumps({"device_type": "ghost", "micro_batch": 1, "seq_length": 1, "hidden": 1,
                             "fwd_ms": 1.0, "bwd_ms": 2.0}))
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("cfg", ["C0", "C1", "C2u"])
def test_cli_plan_with_profiles(tmp_path, cfg):
    """`plan --profiles` (calibration, cli.cpp:107-114, then search): the
    drop-in CLI equals the reference CLI byte for byte, and the Python path
    (calibrate.calibrate_docs + planner.search) finds the same plan."""
    from paper_2405_16256_b200 import abi, calibrate, planner
    _need(PLAN_B200)
    _need(PLAN_REF)
    docs = configs.config(cfg, full=False)
    rng = random.Random(sum(map(ord, cfg)))
    text = _profiles(rng, [g["name"] for g in docs["cluster"]["groups"]])
    paths = _write_inputs(str(tmp_path), docs)
    paths["profiles"] = str(tmp_path / "profiles.ndjson")
    open(paths["profiles"], "w").write(text)
    got = _run_plan(PLAN_B200, paths, str(tmp_path / "b200"))
    want = _run_plan(PLAN_REF, paths, str(tmp_path / "ref"))
    assert got[0] == want[0] == 0, (got[2], want[2])
    assert got[2] == want[2] and "calibration" in want[2]
    for k in want[3]:
        assert got[3][k] == want[3][k], (cfg, k)
    cal, diags = calibrate.calibrate_docs(docs, text)
    assert [d for d in diags] == [line for line in want[2].splitlines() if line]
    out = planner.search(cal)
    p = abi.Problem(cal)
    ref_plan = json.loads(want[3]["plan.json"])
    assert abi.encode_plan(p.group_names, p.plan_from_doc(out.plan)) == abi.encode_plan(
        p.group_names, p.plan_from_doc(ref_plan))
