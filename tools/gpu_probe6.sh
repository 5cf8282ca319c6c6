for v in "" tc_8_256_3 tc_8_256_4 tc_4_512_2 tc_4_512_1; do
  if [ -z "$v" ]; then lib=""; else lib="SK_LIB_PATH=$PWD/tools/ab/$v.so"; fi
  echo "== $v $(env $lib python tools/prof_step.py C5 2 2>&1 | tail -1 | cut -c1-130)"
done
