for c in c5 c2 c3; do
  bash tools/ab_env.sh TMB_WARENA 2 --config $c
done
