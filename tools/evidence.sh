#!/bin/bash
# Round-end evidence on one GPU box: bench lines (c4 with CPU baseline and
# e2e, the reference arm, c1/c2/c3/c5), the ncu launch list of the bench's
# timed region (one step; bench.py brackets it with cudaProfilerStart/Stop), smoke() and the full-size c4 parity check.  Usage (under gpurun):
#   bash tools/evidence.sh TAG      -> gpurun_out/TAG_*
set -u
T=${1:-rXX}
O=gpurun_out
mkdir -p $O
timeout -s KILL 900 python bench.py > $O/${T}_bench_c4.jsonl 2> $O/${T}_bench_c4.err
timeout -s KILL 600 python bench.py --impl reference >> $O/${T}_bench_c4.jsonl 2>> $O/${T}_bench_c4.err
: > $O/${T}_bench_configs.jsonl
for c in c1 c2 c3 c5; do
  timeout -s KILL 900 python bench.py --config $c --steps 10 --warmup 3 >> $O/${T}_bench_configs.jsonl 2>> $O/${T}_bench_configs.err
done
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/${T}_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > $O/${T}_ncu.log 2>&1
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1
timeout -s KILL 900 python tools/validate_full.py > $O/${T}_validate_full_c4.json 2> $O/${T}_validate.err
# one forward wave and one adjoint wave of the headline store, ncu --set full
for k in fwd_tc_kernel adj_tc_kernel; do
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:$k -c 1 -f -o $O/${T}_ncu_$k python tools/prof_run.py > $O/${T}_ncu_$k.log 2>&1
done
tail -n 2 $O/${T}_smoke.log
cut -c1-160 $O/${T}_bench_c4.jsonl $O/${T}_bench_configs.jsonl
# config 5: the K3W batched forward and the adjoint GEMM on the W arena, ncu --set full
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:fwd_k3w -c 1 -f -o $O/${T}_ncu_c5_k3w python tools/prof_run.py --config c5 > $O/${T}_ncu_c5_k3w.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:fwd_tc_kernel -c 1 -f -o $O/${T}_ncu_c5_adjgemm python tools/prof_run.py --config c5 > $O/${T}_ncu_c5_adjgemm.log 2>&1
