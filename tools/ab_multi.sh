#!/bin/bash
# Same-box A/B/C... timing of in-tree library variants libtuckmat_b200_<v>.so:
#   tools/ab_multi.sh "a b c" [rounds] [bench args...]
V=$1; R=${2:-2}; shift; shift
for r in $(seq 1 $R); do
  for v in $V; do
    TMB_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
  done
done
