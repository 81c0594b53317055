# Ring-fed fused FFN (one TMA stream per CTA): quick guarded check, GPU tests, same-call A/B, timelines.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASCADE_FFN_RING=1 timeout -s KILL 240 python -m pytest tests/test_gpu_tiny.py -x -q > gpurun_out/pytest_ring_quick.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_ring_quick.txt
if [ $rc -ne 0 ]; then exit 0; fi
CASCADE_FFN_RING=1 timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ring.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ring.txt
ARMS="ring:CASCADE_FFN_RING=1;warps:X=1" REPS=2 TAG=ring_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="ring:CASCADE_FFN_RING=1;warps:X=1" REPS=2 TAG=ring_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
CASCADE_FFN_RING=1 timeout 600 python scripts/cta_timeline.py mixtral 0,8 ring > gpurun_out/tl_mixtral_ring.txt 2>&1
CASCADE_FFN_RING=1 timeout 600 python scripts/cta_timeline.py olmoe 0,8 ring > gpurun_out/tl_olmoe_ring.txt 2>&1
