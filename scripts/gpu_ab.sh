# A/B pass: GPU parity tests, bench of the default path and of the $ARM_B env variant, ncu launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 300 python -m pytest tests/test_gpu_tiny.py -x -q -k "weights or teacher" > gpurun_out/pytest_quick_$TAG.txt 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
if [ -n "$ARM_B" ]; then
env $ARM_B timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_b.json 2> gpurun_out/bench_${TAG}_b.err
fi
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/profile_step.py --ks 0,8 > gpurun_out/prof_launch_$TAG.log 2>&1
fi
