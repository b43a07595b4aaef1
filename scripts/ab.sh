#!/bin/bash
# A/B the bench on one box: [ROUNDS=n] scripts/ab.sh <libA.so> <libB.so> [libC.so ...]
# (alternates the builds so clock / power-cap drift affects all alike)
N=${ROUNDS:-2}
for i in $(seq 1 $N); do
  for v in "$@"; do
    PARL_LIB=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_classes']
print('$v'.split('/')[-1], round(d['value']), round(d['ms_per_step'],2), 'MHz', d['clocks']['sm_mhz'], {c: round(v['ms_per_step'],2) for c, v in k.items()})"
  done
done
