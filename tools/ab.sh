#!/bin/bash
# A/B timing of in-tree library builds (libtuckmat_b200_a.so / _b.so, or the
# variants listed in $VARIANTS) on the same box, alternating:
#   tools/ab.sh [rounds] [bench args...]
R=${1:-2}; shift
for r in $(seq 1 $R); do
  for v in ${VARIANTS:-a b}; do
    TMB_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
  done
done
