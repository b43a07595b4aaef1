#!/bin/bash
# Strong scaling of C3 (Qwen2.5-7B-shaped tri-model, 1k prompt + 16 x 4k responses, T=66,560 per
# group) to BASELINE.md §4's protocol: a fixed global batch of 16 prompt groups per step, prompt
# groups sharded over N = 1, 2, 4 GPUs of one box (one process per GPU, NCCL over NVLink).
# One JSON line per N in gpurun_out/scale_c3.jsonl.
#   gpurun --gpus 4 -- bash scripts/scale_c3.sh [steps] [warmup]
STEPS=${1:-3}; WARM=${2:-3}
OUT=gpurun_out/scale_c3.jsonl
: > $OUT
for N in 4 2 1; do
  if [ $N -eq 1 ]; then
    python bench.py --config c3 --steps $STEPS --warmup $WARM --no-cpu 2> gpurun_out/scale_c3_n1.err | tail -1 >> $OUT
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29530 + N)) bench.py --config c3 --gpus $N --steps $STEPS --warmup $WARM --no-cpu \
      2> gpurun_out/scale_c3_n$N.err | tail -1 >> $OUT
  fi
done
cat $OUT
