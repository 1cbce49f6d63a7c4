#!/bin/bash
# usage: tools/sweep_ctas.sh NGPUS "ctas list" [extra bench args]
n=$1; shift; list=$1; shift
for c in $list; do
  FTAR_CTAS=$c timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --no-e2e --no-nccl "$@" 2>>gpurun_out/sweep.err > gpurun_out/sw_$c.json
  python -c "import json; d=json.load(open('gpurun_out/sw_$c.json')); print('ctas=$c', '$*', d['value'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['phases_us_rank0'])"
done
