for r in 1 2; do for v in 0 1; do
TMB_FWD_NOSPLIT=$v timeout -s KILL 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nosplit=$v', d['value'], d['forward_ms'], d['adjoint_ms'], d['clocks']['sm_mhz'])"
done; done
