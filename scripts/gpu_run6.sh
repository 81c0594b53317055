cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu6.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu6.txt
timeout 300 python scripts/diag_t.py tiny 3 > gpurun_out/diag6_t3.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err
echo "bench rc=$?" >> gpurun_out/bench6.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches6.csv python scripts/profile_step.py --ks 0,8 > gpurun_out/prof6.log 2>&1
