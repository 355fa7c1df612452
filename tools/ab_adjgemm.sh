# same-box A/B: the adjoint GEMM on the W arena (TMB_ADJ_GEMM=1) vs the consumer-warp adjoint (0)
for c in c5 c2 c3; do
  bash tools/ab_env.sh TMB_ADJ_GEMM 2 --config $c
done
