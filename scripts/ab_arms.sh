# Interleaved A/B of env-variable arms of bench.py in ONE gpurun call (the
# box-to-box spread of a few percent hides small effects; only same-call
# interleaved runs count).  ARMS="name:ENV=v ENV2=w;name2:..."  REPS=n
# CONFIG=mixtral  TAG=x.  Output: gpurun_out/ab/$TAG/<name>_<rep>.json
cd $GRAFT_REPO_ROOT
TAG=${TAG:-ab}
REPS=${REPS:-2}
CONFIG=${CONFIG:-mixtral}
STEPS=${STEPS:-5}
OUT=gpurun_out/ab/$TAG
mkdir -p $OUT
IFS=';' read -ra A <<< "$ARMS"
for r in $(seq 1 $REPS); do
  for arm in "${A[@]}"; do
    name=${arm%%:*}
    envs=${arm#*:}
    env $envs timeout 600 python bench.py --config $CONFIG --steps $STEPS --warmup 3 --no-cpu-baseline \
      > $OUT/${name}_$r.json 2> $OUT/${name}_$r.err
  done
done
python - "$OUT" <<'PY'
import json, os, sys, collections
d = sys.argv[1]
res = collections.defaultdict(list)
for f in sorted(os.listdir(d)):
    if f.endswith(".json"):
        try:
            j = json.load(open(os.path.join(d, f)))
            res[f.rsplit("_", 1)[0]].append(j)
        except Exception:
            pass
with open(os.path.join(d, "summary.txt"), "w") as out:
    for name, js in res.items():
        vals = [j["value"] for j in js]
        ks = {k: [j["per_k"][k]["latency_us"] for j in js] for k in js[0]["per_k"]}
        line = f"{name:10s} mean {sum(vals)/len(vals):9.1f}  runs {vals}  " + " ".join(
            f"K{k}={sum(v)/len(v):.0f}" for k, v in ks.items())
        print(line)
        out.write(line + "\n")
PY
