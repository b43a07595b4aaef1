#!/bin/bash
# One round's bench lines and ncu evidence on one B200 (gpurun -- bash scripts/profile_round.sh TAG).
# Everything lands in gpurun_out/TAG_*; summarise into profiles/ with scripts/ncu_summary.py /
# scripts/traffic.py.  Each ncu capture runs only after the same command exited 0 without ncu.
TAG=${1:-r02}
O=gpurun_out
S=/tmp/prof_$TAG  # .ncu-rep files stay on the box (gpurun_out/ comes back only under 64 MiB)
mkdir -p $S
set -x
python -m pytest tests/test_gpu_c2_invariants.py -q -m gpu -s > $O/${TAG}_c2_invariants.log 2>&1
# bench lines: C2 headline (ours, reference arm), the same-config C1 pairing
python bench.py > $O/${TAG}_bench_c2.json 2> $O/${TAG}_bench_c2.err
python bench.py --impl reference > $O/${TAG}_bench_c2_ref.json 2> $O/${TAG}_bench_c2_ref.err
python bench.py --config c1 > $O/${TAG}_bench_c1.json 2> $O/${TAG}_bench_c1.err
python bench.py --config c1 --impl reference > $O/${TAG}_bench_c1_ref.json 2> $O/${TAG}_bench_c1_ref.err
# K1 / K7 at the stress size
python scripts/stress_k1_k7.py > $O/${TAG}_stress.json 2> $O/${TAG}_stress.err
# launch list + DRAM bytes of one C2 step (8 groups = 2 packed micro-steps)
python bench.py --launch-list --groups 8 --no-cpu > /dev/null 2>&1 && \
ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $O/${TAG}_launches.csv python bench.py --launch-list --groups 8 --no-cpu \
    > $O/${TAG}_launches.log 2>&1
# full captures of the dominant kernels inside a C2 step
for K in "k_gemm_tc2" "k_gemm_group2" "k_attn_fwd_pair" "k_attn_bwd2" "k_ln_bwd_rows4_cs" "k_layernorm4_multi" \
         "k_softmax_bwd_v8"; do
  ncu --set full --clock-control none --import-source on --nvtx --nvtx-include step/ -k regex:"$K" -c 1 \
      -o $S/${TAG}_full_$K python bench.py --launch-list --groups 4 --no-cpu > $O/${TAG}_full_$K.log 2>&1
done
# the head GEMM (the policy's full-vocabulary logits: the largest k_gemm_tc2 launch)
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include step/ --kernel-name-base demangled -k regex:"k_gemm_tc2<\\(int\\)0, \\(int\\)0, \\(int\\)1, \\(int\\)256>" \
    -c 1 -o $S/${TAG}_full_head_gemm python bench.py --launch-list --groups 4 --no-cpu > $O/${TAG}_full_head.log 2>&1
# K1 / K7 at the stress size
ncu --set full --clock-control none --import-source on -k regex:"k_grpo_tokens" -c 1 -o $S/${TAG}_full_k7_stress \
    python scripts/stress_k1_k7.py --only k7 --reps 1 > $O/${TAG}_full_k7.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pack" -c 1 -o $S/${TAG}_full_k1_stress \
    python scripts/stress_k1_k7.py --only k1 --reps 1 > $O/${TAG}_full_k1.log 2>&1
# summaries (and the raw counter pages) of every capture
for R in $S/*.ncu-rep; do
  B=$(basename $R .ncu-rep)
  python scripts/ncu_summary.py report $R > $O/$B.md 2>&1
  ncu -i $R --page raw --csv > $O/$B.raw.csv 2>/dev/null
done
python scripts/ncu_summary.py launches $O/${TAG}_launches.csv > $O/${TAG}_c2_launches.md 2>&1
python scripts/traffic.py $O/${TAG}_launches.csv > $O/${TAG}_traffic.json 2>&1
ls -la $O $S
