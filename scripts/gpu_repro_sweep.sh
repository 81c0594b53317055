# Repeat the two-session device scenario sweep test to reproduce a rare failure (cell errors are named now).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in $(seq 1 12); do
  timeout -s KILL 300 python -m pytest tests/test_gpu_interop.py -q -k two_sessions > gpurun_out/sweep_rep_$i.txt 2>&1; echo "rc=$?" >> gpurun_out/sweep_rep_$i.txt
done
grep -h "rc=\|failed:" gpurun_out/sweep_rep_*.txt | sort | uniq -c > gpurun_out/sweep_rep_summary.txt
