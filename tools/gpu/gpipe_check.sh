#!/bin/bash
# GPipe evaluator: parity tests and the GPipe-at-scale search time
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_evaluate.py tests/test_gpu_log.py -q -p no:cacheprovider -k "not per_pp and not c3_full" > gpurun_out/pytest_gpipe.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpipe.log
python - > gpurun_out/gpipe_run.txt 2>&1 <<'PY'
import json, time, sys
sys.path.insert(0, ".")
from paper_2405_16256_b200 import planner
d = json.load(open("tests/golden/gpipe_scale.json"))["docs"]
for _ in range(3):
    t0 = time.time(); o = planner.search(d); print(json.dumps({"wall_s": time.time() - t0, "dev_ms": o.device_ms, "sim": o.candidates_simulated}))
PY
