# same-box A/B: the adjoint GEMM's split final wave (TMB_ADJ_NOSPLIT=0) vs unsplit (1)
for c in c2 c3 c5; do
  bash tools/ab_env.sh TMB_ADJ_NOSPLIT 2 --config $c
done
