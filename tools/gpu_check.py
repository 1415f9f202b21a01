"""Dev check: GPU search vs the C oracle on small configs, plus timings."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port
from paper_2405_16256_b200 import configs, abi, planner

def run(name, cfg, check=True, timed=False):
    P = abi.Problem(cfg)
    eng = planner.engine(0)
    import ctypes as C
    opts = abi.hp_search_opts(0, 1, 0, abi.HP_FLAG_TIME_KERNELS if timed else 0, 0.0)
    r = abi.hp_result()
    t0 = time.time(); st = eng._lib.hp_search(eng._ctx, P.ptr(), C.byref(opts), C.byref(r)); t1 = time.time()
    assert st == 0, (st, eng._lib.hp_last_error(eng._ctx))
    line = {"cfg": name, "gpu_s": round(t1 - t0, 4), "dev_ms": round(r.device_ms, 2), "sim": r.candidates_simulated,
            "pruned": r.candidates_pruned, "time": r.best_time_s, "launches": r.gpu_launches,
            "enc": abi.encode_plan(P.group_names, r.best_plan), "iters": r.hill_iterations, "host_ms": round(r.host_ms, 1),
            "eval_ms": round(r.eval_ms, 2), "eval_launches": r.eval_launches, "fp64_ops": r.eval_fp64_ops,
            "h2d": r.h2d_bytes, "d2h": r.d2h_bytes}
    if r.eval_ms > 0: line["eval_tflops"] = round(r.eval_fp64_ops / r.eval_ms / 1e9, 3)
    if check:
        t0 = time.time(); st, o = port.search(P); t1 = time.time()
        line["oracle_s"] = round(t1 - t0, 3)
        line["match"] = (o.best_time_s == r.best_time_s and o.candidates_simulated == r.candidates_simulated and
                         o.candidates_pruned == r.candidates_pruned and
                         abi.encode_plan(P.group_names, o.best_plan) == line["enc"])
        if not line["match"]:
            line["oracle"] = [o.candidates_simulated, o.candidates_pruned, o.best_time_s, abi.encode_plan(P.group_names, o.best_plan)]
    print(json.dumps(line), flush=True)

which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "small":
    for n in ["C0", "C1", "C2u", "C2"]:
        run(n, configs.config(n, full=True))
    run("C3pp12", configs.with_pp(configs.config("C3", full=True), [12]))
    run("C3pp24", configs.with_pp(configs.config("C3", full=True), [24]))
    c = configs.config("C5"); c["planner"]["pipeline_degrees"] = [3]; c["planner"]["micro_batch_candidates"] = [8]
    run("C5pp3B8", c)
if which in ("small", "c3"):
    for i in range(2):
        run("C3full", configs.config("C3", full=True), check=False)
    run("C3full_timed", configs.config("C3", full=True), check=False, timed=True)
if which in ("small", "peak"):
    import ctypes as C
    from paper_2405_16256_b200._lib import lib
    l = lib(); l.hp_fp64_peak.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    a, m = C.c_double(), C.c_double()
    l.hp_fp64_peak(0, C.byref(a), C.byref(m))
    print(json.dumps({"fp64_dadd_ops_per_s": a.value, "fp64_mix_ops_per_s": m.value}))
if which in ("default",):
    from oracle import ref
    for n in ["C0", "C1", "C2u", "C2", "C3"]:
        cfg = configs.config(n, full=False)
        P = abi.Problem(cfg)
        eng = planner.engine(0)
        t0 = time.time(); r = eng.search_shard(P); t1 = time.time()
        rr = ref.search(cfg, jobs=os.cpu_count())
        enc = abi.encode_plan(P.group_names, r.best_plan)
        renc = abi.encode_plan(P.group_names, P.plan_from_doc(rr["plan"]))
        line = {"cfg": n + "-default", "gpu_s": round(t1 - t0, 4), "dev_ms": round(r.device_ms, 2),
                "sim": r.candidates_simulated, "pruned": r.candidates_pruned, "time": r.best_time_s,
                "gb": r.global_bound, "ref_s": rr["wall_s"],
                "match": (rr["candidates_simulated"] == r.candidates_simulated and
                          rr["candidates_pruned"] == r.candidates_pruned and
                          rr["eval"]["iteration_time_s"] == r.best_time_s and renc == enc)}
        if not line["match"]:
            line["ref"] = [rr["candidates_simulated"], rr["candidates_pruned"], rr["eval"]["iteration_time_s"], renc, enc]
        print(json.dumps(line), flush=True)
if which in ("c5",):
    c = configs.config("C5"); c["model"]["num_layers"] = 40
    run("C5-L40", c)
    c = configs.config("C5"); c["model"]["num_layers"] = 40; c["planner"]["schedule"] = "gpipe"
    for g in c["cluster"]["groups"]: g["memory_bytes"] = 400e9
    run("C5-L40-gpipe", c)
    c = configs.config("C5"); c["planner"]["pipeline_degrees"] = [3]; c["planner"]["micro_batch_candidates"] = [1]
    run("C5pp3B1", c, check=False)
    run("C5", configs.config("C5"), check=False, timed=True)
