for r in 1 2; do for c in 24 48 96 12; do
TMB_TC_CHAIN=$c timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chain $c', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
done; done
