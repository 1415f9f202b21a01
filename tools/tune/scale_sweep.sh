#!/bin/bash
# A/B of climb scheduling knobs on the sharded C3 sweep (run on a 4-GPU box):
#   gpurun --gpus 4 -- 'bash tools/tune/scale_sweep.sh "4 X=0" "4 HP_CRIT_SMS=0" "2 HP_R1_THR=74" ...'
mkdir -p gpurun_out
run() { n=$1; shift; env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('n=$n $*', round(d['ms_per_step'],1), [round(x,1) for x in d['config']['rank_device_ms']])"; }
for spec in "$@"; do run $spec; done
