# Large seeded fuzz sweeps (GPU): python scripts/fuzz_big.py SEED
# 300 fast==exact kernel cases and 80 sslic_segment-vs-oracle cases.
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_gpu_fast as t
import paper_1806_08741_b200 as s
fails = 0
cases = t._fuzz_cases(n=300, seed=int(sys.argv[1]))
for i, c in enumerate(cases):
    try:
        t.test_fast_equals_exact_fuzz.__wrapped__(s, c) if hasattr(t.test_fast_equals_exact_fuzz, "__wrapped__") else t.test_fast_equals_exact_fuzz(s, c)
    except Exception as e:
        fails += 1
        print("FAIL", i, c, repr(e)[:200])
print("done", len(cases), "fails", fails)

# the whole pipeline against the CPU oracle
import test_gpu_parity as tp
import oracle
oracle.build()
o = oracle.Oracle()
pf = 0
pcases = tp._pipeline_fuzz(n=80, seed=int(sys.argv[1]) + 1)
for i, c in enumerate(pcases):
    try:
        tp.test_segment_matches_oracle_fuzz(s, o, c)
    except Exception as e:
        pf += 1
        print("PIPE FAIL", i, c, repr(e)[:200])
print("pipeline done", len(pcases), "fails", pf)
