#!/bin/bash
# Same-box A/B matrix of library variants (libtuckmat_b200_<v>.so, TMB_LIB_VARIANT) x
# TMB_TC_DEBUG settings: VDS="a:0 b:0 b:16" bash tools/ab_fold.sh
for r in 1 2; do
for vd in ${VDS:-a:0 d:0 a:16 d:16 d:48}; do
v=${vd%%:*}; dbg=${vd##*:}
TMB_TC_DEBUG=$dbg TMB_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v dbg=$dbg', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
done; done
