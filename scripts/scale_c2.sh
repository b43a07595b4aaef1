#!/bin/bash
# Strong scaling to BASELINE.md §4's protocol: C2, a fixed global batch of 64 prompt groups per
# step split over N = 1, 2, 4 GPUs of one box (one process per GPU, NCCL over NVLink), each rank
# packing PACK groups per sequence.  One JSON line per N in gpurun_out/scale_c2.jsonl.
#   gpurun --gpus 4 -- bash scripts/scale_c2.sh [steps] [warmup] [pack]
STEPS=${1:-5}; WARM=${2:-3}; PACK=${3:-4}
OUT=gpurun_out/scale_c2.jsonl
: > $OUT
python bench.py --steps $STEPS --warmup $WARM --pack $PACK --no-cpu 2> gpurun_out/scale_n1.err | tail -1 >> $OUT
for N in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29510 + N)) \
    bench.py --gpus $N --steps $STEPS --warmup $WARM --pack $PACK --no-cpu 2> gpurun_out/scale_n$N.err | tail -1 >> $OUT
done
cat $OUT
