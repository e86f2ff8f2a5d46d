#!/bin/bash
# Control-flow rehearsal of the N > 1 bench on a one-GPU box: gloo, every rank on GPU 0 (FM_BENCH_DRYRUN_GLOO).
# Not a measurement: checks that shard -> launch -> pack -> gather -> unshard, the weak companion, the e2e leg and
# the reference arm run to a JSON line at N = 2 / 4 / 8 exactly as the driver launches them.
export FM_BENCH_DRYRUN_GLOO=1
for n in 2 8; do
  timeout 600 python bench.py --gpus $n --steps 16 --warmup 3 --e2e-steps 2 > gpurun_out/dry_n$n.json 2> gpurun_out/dry_n$n.err; echo "spawn n=$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 --steps 16 --warmup 3 --e2e-steps 2 > gpurun_out/dry_n4.json 2> gpurun_out/dry_n4.err; echo "torchrun n=4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/dry_ref_n2.json 2> gpurun_out/dry_ref_n2.err; echo "torchrun ref n=2 rc=$?"
