cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -s -x > gpurun_out/pytest_gpu3.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
echo "bench rc=$?" >> gpurun_out/bench3.err
