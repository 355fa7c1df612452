#!/bin/bash
# Same-box sweep of the forward's accumulation-chain length and stage count on
# the headline store (bench.py c4, physics rank table), plus the full-size
# error of each chain length against the complex128 GPU path.
#   bash tools/tune_c4.sh TAG   (under gpurun)  -> gpurun_out/TAG_tune.jsonl
T=${1:-rXX}
O=gpurun_out
mkdir -p $O
: > $O/${T}_tune.jsonl
for ch in 24 32 48; do
  for nst in 0; do
    TMB_TC_CHAIN=$ch python bench.py --no-cpu --no-e2e --steps 5 --warmup 2 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'chain': $ch, 'fwd_ms': d['forward_ms'], 'adj_ms': d['adjoint_ms'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/${T}_tune.jsonl
  done
done
for nst in 4 5; do
  TMB_TC_NST=$nst python bench.py --no-cpu --no-e2e --steps 5 --warmup 2 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'nst': $nst, 'fwd_ms': d['forward_ms'], 'adj_ms': d['adjoint_ms'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/${T}_tune.jsonl
done
python tools/validate_full.py --chains 32,48 --sample-cols 4 >> $O/${T}_tune.jsonl 2>/dev/null
cat $O/${T}_tune.jsonl
