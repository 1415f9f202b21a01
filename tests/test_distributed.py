"""Multi-process (world_size 2, gloo on CPU) path of the sharded search:
disjoint leaf shards per rank, one all-gather of the fixed-size per-rank
records, identical exact reduction on every rank. The per-rank search is the
CPU emulation of the device decomposition (tests/emu) so this runs without a
GPU; on the B200 box the same planner.search_sharded drives the CUDA engine
over NCCL (tests/test_gpu_*)."""
from __future__ import annotations

import ctypes as C
import json
import os
import socket
import struct

import torch.multiprocessing as mp

from conftest import ROOT, build_emu, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, names, out_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2405_16256_b200 import abi, planner
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    emu = build_emu()

    def shard_fn(p, r, w, bound):
        res = abi.hp_result()
        assert emu.emu_search_shard(C.byref(p.struct), r, w, C.byref(res)) == abi.HP_OK
        return res

    cases = {c["name"]: c for c in load_golden("search_cases.json")}
    results = {}
    for n in names:
        out = planner.search_sharded(cases[n]["docs"], rank, world, None, shard_fn=shard_fn)
        results[n] = [out.iteration_time_s.hex(), out.candidates_simulated, out.candidates_pruned,
                      json.dumps(out.plan, sort_keys=True)]
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump(results, f)
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_search(tmp_path):
    cases = [c for c in load_golden("search_cases.json")
             if c["status"] == 0 and not c["docs"]["planner"].get("time_bound_pruning", True)]
    names = [c["name"] for c in cases[:12]]
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(2, _free_port(), names, out), nprocs=2, join=True, start_method="spawn")
    r0 = json.load(open(out + ".0"))
    r1 = json.load(open(out + ".1"))
    assert r0 == r1  # every rank reduces to the same plan
    by = {c["name"]: c for c in cases}
    for n in names:
        t_hex, sim, pr, plan = r0[n]
        assert float.fromhex(t_hex) == by[n]["iteration_time_s"]
        assert struct.pack(">d", float.fromhex(t_hex)).hex() == by[n]["iteration_bits"]
        assert (sim, pr) == (by[n]["candidates_simulated"], by[n]["candidates_pruned"])
        want = dict(by[n]["plan"])
        got = json.loads(plan)
        assert got["stages"] == want["stages"]
        assert got["micro_batches_per_dp_replica"] == want["micro_batches_per_dp_replica"]
