# c5 adjoint: right-hand-side groups (default NR = 4) vs the single-RHS kernel per rhs (TMB_ADJ_NR1=1)
for r in 1 2; do for v in 0 1; do
TMB_ADJ_NR1=$v timeout -s KILL 300 python bench.py --config c5 --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMB_ADJ_NR1=$v', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
done; done
