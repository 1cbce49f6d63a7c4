# Round-end measurement set (run on a 4-GPU box: bash tools/final_runs.sh [outdir])
set -u
O=${1:-gpurun_out/final3}; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --impl reference > $O/ref1.json 2> $O/ref1.err; echo ref1=$?
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py > $O/b1.json 2> $O/b1.err; echo b1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29621 bench.py --impl reference --gpus 2 > $O/ref2.json 2> $O/ref2.err; echo ref2=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29622 bench.py --gpus 2 > $O/b2.json 2> $O/b2.err; echo b2=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29623 bench.py --impl reference --gpus 4 > $O/ref4.json 2> $O/ref4.err; echo ref4=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29624 bench.py --gpus 4 > $O/b4.json 2> $O/b4.err; echo b4=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29625 tools/sweep.py > $O/sweep2.jsonl 2> $O/sweep2.err; echo s2=$?
timeout 600 $TR --nproc-per-node 4 --master-port 29626 tools/sweep.py > $O/sweep4.jsonl 2> $O/sweep4.err; echo s4=$?
timeout 600 $TR --nproc-per-node 4 --master-port 29627 tools/bench_catchup.py --stripe --ctas 8,16,32,64 > $O/catchup4.jsonl 2> $O/catchup4.err; echo c4=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29628 tools/hsdp_churn.py > $O/churn4.json 2> $O/churn4.err; echo ch4=$?
timeout 300 $TR --nproc-per-node 3 --master-port 29629 tools/hsdp_churn.py --steps 10 --kill-at 3 --dead 3 > $O/churn3kat.json 2> $O/churn3kat.err; echo ch3=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29630 tools/intra_bench.py > $O/intra4.jsonl 2> $O/intra4.err; echo i4=$?
