#!/bin/bash
# bench.py --gpus N under torchrun with all ranks time-sliced on the one GPU
# gpurun offers (PF_BENCH_SHARE_GPU=1): exercises the N > 1 bench path end to
# end (sharding, IPC exchange, consistency check, e2e); the numbers are NOT
# scaling numbers.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CFG=${CFG:-cfg1}
for N in ${NS:-2 4}; do
  PF_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps ${STEPS:-100} --warmup 3 \
    --config $CFG > gpurun_out/shared_n$N.json 2> gpurun_out/shared_n$N.log
  echo "N=$N rc=$?"; tail -c 1500 gpurun_out/shared_n$N.json
done
