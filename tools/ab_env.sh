#!/bin/bash
# A/B timing of an environment switch on the same box, alternating 0 / $AB_VAL (default 1):
#   tools/ab_env.sh VAR [rounds] [bench args...]
V=${1:-TMB_FWD_NOSPLIT}; R=${2:-2}; shift; shift
for r in $(seq 1 $R); do for v in 0 1; do
env $V=$((v * ${AB_VAL:-1})) timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$V=$v', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
done; done
