# Quick GPU pass: parity tests, smoke, one bench line (our arm).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-chk}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$TAG.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.txt
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
