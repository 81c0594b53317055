cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu2.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo "bench rc=$?" >> gpurun_out/bench2.err
