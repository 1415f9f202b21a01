#!/bin/bash
# per-leaf step timeline of one shard of an N-GPU C3 sweep, run alone on one GPU
# usage: SHARD=0/2 bash tools/gpu/trace_shard.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
S=${SHARD:-0/2}
tag=$(echo $S | tr / _)
RUN_SHARD=$S python tools/run_search.py C3 full 2 > gpurun_out/shard_$tag.txt 2>&1
RUN_SHARD=$S HP_DEBUG_TRACE=gpurun_out/trace_$tag.bin python tools/run_search.py C3 full 1 >> gpurun_out/shard_$tag.txt 2>&1
python tools/analysis/leaf_timeline.py gpurun_out/trace_$tag.bin 6 >> gpurun_out/shard_$tag.txt 2>&1
rm -f gpurun_out/trace_$tag.bin
