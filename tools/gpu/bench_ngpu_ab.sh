#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
port=29600
for v in ${AB_VARIANTS:-"HP_X=0" "HP_NO_LAT=1"}; do
  port=$((port+1))
  env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab_$port.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v', d['ms_per_step'], d['config']['rank_device_ms'])" >> gpurun_out/scale_ab_n$N.txt
done
