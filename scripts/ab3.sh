# A/B/C of env-selected kernel variants on a bench config (alternating, 2 rounds each).
# usage: bash scripts/ab3.sh TAG "ENV_A" "ENV_B" "ENV_C" [bench args]
cd $GRAFT_REPO_ROOT
T=$1; A=$2; B=$3; Cc=$4; shift 4
for r in 1 2; do
  for v in A B C; do
    if [ $v = A ]; then E="$A"; elif [ $v = B ]; then E="$B"; else E="$Cc"; fi
    env $E timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e "$@" > gpurun_out/${T}_${v}${r}.log 2>&1
  done
done
python - "$T" <<'PY'
import json, sys, glob
t = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{t}_[ABC][12].log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            print(f, round(d["value"] / 1e9, 2), "Gvox/s frac", round(r["frac"], 4),
                  "evals", round(r["algorithmic"]["evals_performed_per_voxel"][-1], 3),
                  "ms/it", [round(x, 2) for x in r["kernel_ms_per_iteration"]])
PY
