"""The C-ABI boundary (include/hetplan_b200.h): the in-tree library loads
without a GPU, exports every declared entry point, its struct layout matches
the ctypes mirror, and host-side validation / ordering behave like the
reference (ConfigError messages of types.cpp:78-163, planner.cpp:600-607;
better_than of planner.cpp:178-200). No compute calls here."""
from __future__ import annotations

import copy
import ctypes as C
import os
import random
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2405_16256_b200 import abi, configs
from paper_2405_16256_b200._lib import EXPORTED, SO, lib

HEADER = os.path.join(ROOT, "include", "hetplan_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    l = lib()
    decl = declared_functions()
    assert set(decl) == set(EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", SO], capture_output=True, text=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for fn in decl:
        assert fn in syms, fn
        assert hasattr(l, fn)
    assert l.hp_abi_version() == 3


def test_struct_layout_matches_header(tmp_path):
    structs = ["hp_model", "hp_group", "hp_link", "hp_cluster", "hp_train", "hp_planner", "hp_problem",
               "hp_stage", "hp_plan", "hp_search_opts", "hp_result", "hp_log_entry", "hp_trace_event",
               "hp_stage_eval", "hp_plan_eval"]
    src = tmp_path / "layout.c"
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for s in structs:
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for name, _ in getattr(abi, s)._fields_:
            lines.append(f'printf("{s}.{name} %zu\\n", offsetof({s}, {name}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True)
               .stdout.splitlines())
    for s in structs:
        cls = getattr(abi, s)
        assert int(got[s]) == C.sizeof(cls), s
        for name, _ in cls._fields_:
            assert int(got[f"{s}.{name}"]) == getattr(cls, name).offset, f"{s}.{name}"


def validate(docs):
    l = lib()
    p = abi.Problem(docs)
    st = l.hp_validate(None, p.ptr())
    return st, (l.hp_last_error(None) or b"").decode()


BAD = [
    ("model", lambda d: d["model"].__setitem__("num_heads", 7), "model: hidden_size must be divisible by num_heads"),
    ("model", lambda d: d["model"].__setitem__("bytes_per_element", 3), "model: bytes_per_element must be 2 or 4"),
    ("model", lambda d: d["model"].__setitem__("num_layers", 0), "model: num_layers must be >= 1"),
    ("cluster", lambda d: d["cluster"]["groups"][1].__setitem__("name", "amd"), "cluster: duplicate group name 'amd'"),
    ("cluster", lambda d: d["cluster"]["groups"][0].__setitem__("compute_efficiency", 1.6),
     "cluster: group 'amd': compute_efficiency must be in (0, 1.5]"),
    ("cluster", lambda d: d["cluster"]["groups"][0].__setitem__("bwd_fwd_ratio", 0.5),
     "cluster: group 'amd': bwd_fwd_ratio must be >= 1"),
    ("cluster", lambda d: d["cluster"]["links"].pop(0), "cluster: group 'amd' needs exactly one intra-node link"),
    ("cluster", lambda d: d["cluster"]["links"][4].__setitem__("efficiency", 1.2), "cluster: link efficiency must be in (0, 1]"),
    ("train", lambda d: d["train"].__setitem__("micro_batch_size", 1000),
     "train: micro_batch_size must not exceed global_batch_size"),
    ("planner", lambda d: d["planner"].__setitem__("memory_headroom", 1.5), "planner: memory_headroom must be in (0, 1]"),
    ("planner", lambda d: d["planner"].__setitem__("pipeline_degrees", [0, 2]), "planner: pipeline degrees must be >= 1"),
    ("planner", lambda d: d["planner"].__setitem__("stage_order_beam_width", -1),
     "planner: stage_order_beam_width must be >= 0"),
    # the unknown name itself is in the message (types.cpp:126)
    ("cluster", lambda d: d["cluster"]["links"][0]["endpoints"].__setitem__("group", "nosuch"),
     "cluster: link references unknown group 'nosuch'"),
    ("cluster", lambda d: d["cluster"]["links"][4]["endpoints"].__setitem__("group_b", "nosuch"),
     "cluster: inter-group link references undeclared group"),
]


@pytest.mark.parametrize("doc,mutate,msg", BAD)
def test_validation_messages(doc, mutate, msg):
    d = copy.deepcopy(configs.config("C0"))
    mutate(d)
    st, err = validate(d)
    assert st == abi.HP_BAD_CONFIG
    assert err == msg
    from oracle import ref
    if ref.available():  # the reference raises the same ConfigError text
        r = ref.search(d)
        assert r["status"] == 1 and r["error"] == msg


def test_long_names_and_many_groups():
    """Group names of any length and up to HP_MAX_GROUPS groups pass the
    boundary; a longer list is rejected with a ConfigError naming the cap."""
    d = copy.deepcopy(configs.config("C0"))
    long_name = "accelerator-with-a-very-long-vendor-specific-name-0123456789"
    for l in d["cluster"]["links"]:
        ep = l["endpoints"]
        for k in ("group", "group_a", "group_b"):
            if ep.get(k) == "amd":
                ep[k] = long_name
    d["cluster"]["groups"][0]["name"] = long_name
    assert validate(d)[0] == abi.HP_OK
    p = abi.Problem(d)
    pl = p.plan_from_doc({"schedule": "1f1b", "micro_batches_per_dp_replica": 4, "micro_batch_size": 1,
                          "stages": [{"layer_range": [0, 80], "group": long_name, "nodes_used": 1,
                                      "tp_degree": 8, "dp_degree": 1}]})
    assert abi.encode_plan(p.group_names, pl).startswith("1f1b|4|1|" + long_name + ":0-80")
    from paper_2405_16256_b200 import configs as cf
    many = [cf.group(f"g{k}", cf.GROUP_PRESETS["amd"], 1, 8) for k in range(abi.HP_MAX_GROUPS)]
    d2 = copy.deepcopy(configs.config("C0"))
    d2["cluster"] = cf.cluster_doc(many)
    assert validate(d2)[0] == abi.HP_OK
    d2["cluster"] = cf.cluster_doc(many + [cf.group("extra", cf.GROUP_PRESETS["amd"], 1, 8)])
    with pytest.raises(abi.ConfigError, match="at most 16 device groups"):
        validate(d2)


def test_valid_config_validates():
    for n in ["C0", "C1", "C2", "C3", "C4:nvidia+amd", "C5"]:
        assert validate(configs.config(n))[0] == abi.HP_OK


def test_better_than_matches_encoding_order():
    """hp_better_than == (time, pp, encode_plan string) lexicographic."""
    rng = random.Random(7)
    docs = configs.config("C0")
    p = abi.Problem(docs)
    l = lib()

    def rand_plan():
        pl = abi.hp_plan()
        pl.schedule = 1
        pl.micro_batches_per_dp_replica = rng.choice([8, 16, 64, 128])
        pl.micro_batch_size = rng.choice([1, 2])
        P = rng.choice([2, 3])
        pl.n_stages = P
        b = 0
        for i in range(P):
            c = rng.choice([9, 10, 11, 100 // P])
            pl.stages[i].layer_begin, pl.stages[i].layer_end = b, b + c
            b += c
            pl.stages[i].group = rng.randrange(2)
            pl.stages[i].tp_degree = rng.choice([1, 8])
            pl.stages[i].dp_degree = 2
            pl.stages[i].nodes_used = rng.choice([1, 2])
        return pl

    for _ in range(300):
        a, b = rand_plan(), rand_plan()
        ta, tb = rng.choice([1.0, 2.0]), rng.choice([1.0, 2.0])
        want = abi.better_key(p.group_names, ta, a.n_stages, a) < abi.better_key(p.group_names, tb, b.n_stages, b)
        got = l.hp_better_than(p.ptr(), ta, C.byref(a), tb, C.byref(b)) < 0
        assert got == want
