for v in "" "SK_REGSOLVE=3" "SK_ODDSPAN_THETA=0" "SK_REGSOLVE=3 SK_ODDSPAN_THETA=0" "SK_THETA_THREADS=448" "SK_THETA_THREADS=384" "SK_REGSOLVE=0"; do
  for rep in 1 2; do
    echo "== [$v] $(env $v python tools/prof_step.py C3 3 2>&1 | tail -1 | cut -c1-120)"
  done
done
