# Ring engine for 9-16 tokens (B slice in the TMA stages, B producer owns the readiness wait): guarded check, tests, A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASCADE_RING_MAXT=16 timeout -s KILL 240 python -m pytest tests/test_gpu_tiny.py -x -q > gpurun_out/pytest_ring3_quick.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_ring3_quick.txt
if [ $rc -ne 0 ]; then exit 0; fi
CASCADE_RING_MAXT=16 timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ring3.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ring3.txt
ARMS="maxt16:CASCADE_RING_MAXT=16;maxt8:X=1" REPS=2 TAG=ring3_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="maxt16:CASCADE_RING_MAXT=16;maxt8:X=1" REPS=2 TAG=ring3_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="maxt16:CASCADE_RING_MAXT=16;maxt8:X=1" REPS=1 TAG=ring3_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
CASCADE_RING_MAXT=16 timeout 600 python scripts/cta_timeline.py mixtral 8 ring3 > gpurun_out/tl_mixtral_ring3.txt 2>&1
