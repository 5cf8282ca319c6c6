timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_all.log 2>&1
for c in C4 C2 C1; do for pc in 1 0 1 0; do echo "== $c pair_chains=$pc $(SK_PAIR_CHAINS=$pc python tools/prof_step.py $c 5 2>&1 | tail -1 | cut -c1-130)"; done; done > gpurun_out/pair_ab.txt 2>&1
