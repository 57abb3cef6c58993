# A/B of kernel variants on the config-3 bench (alternating, 2 rounds each).
# usage: bash scripts/ab.sh TAG "ENV_A" "ENV_B" [bench args]
cd $GRAFT_REPO_ROOT
T=$1; A=$2; B=$3; shift 3
for r in 1 2; do
  for v in A B; do
    if [ $v = A ]; then E="$A"; else E="$B"; fi
    env $E timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/${T}_${v}${r}.log 2>&1
  done
done
python - "$T" <<'PY'
import json, sys, glob
t = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{t}_[AB][12].log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, round(d["value"] / 1e9, 2), "Gvox/s frac", round(r["frac"], 4),
                  "evals", round(r["algorithmic"]["evals_performed_per_voxel"][-1], 3),
                  "redec", r["algorithmic"]["fp64_redecided_voxel_frac"][-1])
PY
