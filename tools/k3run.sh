#!/bin/bash
# K3 batched forward: parity cases, then config-5 forward time at several factor-ring depths vs the x-in-B forward
python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider -k "k3" > gpurun_out/k3.log 2>&1
tail -2 gpurun_out/k3.log
for v in "TMB_K3_JR=3" "TMB_K3_JR=6" "TMB_K3_JR=12" "TMB_K3=0"; do
  env $v python bench.py --config c5 --no-cpu --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['forward_ms'], d['adjoint_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
