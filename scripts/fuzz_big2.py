# Large seeded fuzz sweeps (GPU), part 2: python scripts/fuzz_big2.py SEED
# z-slab splits (summed slab engines == one engine) and pipelined run_slic
# on random >= 2^24-voxel geometries (pinned == pageable).
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_fast as t
import paper_1806_08741_b200 as s
seed = int(sys.argv[1])
for name, gen, fn, n in [("slabs", t._slab_fuzz, t.test_slab_engines_fuzz, 80),
                         ("pipelined", t._pipeline_geoms, t.test_run_slic_pipelined_random_geometry, 16)]:
    fails = 0
    cases = gen(n=n, seed=seed)
    for i, c in enumerate(cases):
        try:
            fn(s, c)
        except Exception as e:
            fails += 1
            print(name, "FAIL", i, c, repr(e)[:200])
    print(name, "done", len(cases), "fails", fails, flush=True)
