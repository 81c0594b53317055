# Runs the quick parity tests, then bench.py once per arm (env strings in ARMS, ';'-separated).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-arms}
timeout 300 python -m pytest tests/test_gpu_tiny.py -x -q -k "weights or teacher" > gpurun_out/pytest_quick_$TAG.txt 2>&1 || exit 1
if [ -n "$FULL_TESTS" ]; then
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
fi
i=0
IFS=';' read -ra A <<< "$ARMS"
for arm in "${A[@]}"; do
  env $arm timeout 900 python bench.py --steps ${STEPS:-4} --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2> gpurun_out/bench_${TAG}_$i.err
  echo "$arm" > gpurun_out/bench_${TAG}_$i.arm
  i=$((i+1))
done
