cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu7.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu7.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err
echo "bench rc=$?" >> gpurun_out/bench7.err
CASCADE_NO_PREFETCH=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_nopf.json 2> gpurun_out/bench7_nopf.err
