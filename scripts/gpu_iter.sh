# Iteration pass: GPU parity tests + per-CTA timelines (+ optional bench)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
for cfg in ${TL_CFGS:-mixtral}; do
  timeout 600 python scripts/cta_timeline.py $cfg ${TL_KS:-0,8} $TAG > gpurun_out/tl_${cfg}_$TAG.txt 2>&1
done
if [ -n "$BENCH" ]; then timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; fi
