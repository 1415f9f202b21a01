mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py -m gpu -x -q -k scheduling > gpurun_out/sw_pytest.log 2>&1; tail -1 gpurun_out/sw_pytest.log
run() { n=$1; shift; env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('n=$n $*', round(d['ms_per_step'],1), [round(x,1) for x in d['config']['rank_device_ms']])"; }
run 4 X=0
run 4 HP_R1_THR=74
run 4 HP_R1_THR=296
run 4 HP_CRIT_SMS=0
run 2 X=0
run 2 HP_CRIT_SMS=74
run 2 HP_R1_THR=74
run 2 HP_R1_THR=296
