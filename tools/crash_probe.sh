for sz in 6000x64 12000x48 4200x40 20000x24 20000x200; do
  SK_THETA_SYM=0 timeout 120 python tools/sym_check.py child /tmp/p_$sz.npz $sz > /tmp/o_$sz.txt 2>&1; echo "pair $sz rc=$?"
  timeout 120 python tools/sym_check.py child /tmp/s_$sz.npz $sz > /tmp/o2_$sz.txt 2>&1; echo "sym $sz rc=$?"
done
