# Robustness evidence: the GPU suite twice (flakiness), once with the register FFN engine everywhere, and
# compute-sanitizer memcheck / racecheck / synccheck on small ring-FFN steps.
cd $GRAFT_REPO_ROOT; O=gpurun_out/robust; mkdir -p $O
for i in 1 2; do timeout -s KILL 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_run$i.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu_run$i.txt; done
CASCADE_FFN_RING=0 timeout -s KILL 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_register_engine.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu_register_engine.txt
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/ring_dbg.py tiny 16 > $O/sanitizer_${tool}_tiny.txt 2>&1; echo "rc=$?" >> $O/sanitizer_${tool}_tiny.txt
done
timeout -s KILL 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/ring_dbg.py mixtral 16 > $O/sanitizer_memcheck_mixtral1L.txt 2>&1; echo "rc=$?" >> $O/sanitizer_memcheck_mixtral1L.txt
