# Ring engine for T <= 8 (default) vs the register engine: GPU tests, same-call A/B on three configs, timelines.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_ring2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ring2.txt
ARMS="ring:X=1;warps:CASCADE_FFN_RING=0" REPS=2 TAG=ring2_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="ring:X=1;warps:CASCADE_FFN_RING=0" REPS=2 TAG=ring2_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="ring:X=1;warps:CASCADE_FFN_RING=0" REPS=2 TAG=ring2_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
timeout 600 python scripts/cta_timeline.py mixtral 0,4,8 ring2 > gpurun_out/tl_mixtral_ring2.txt 2>&1
timeout 600 python scripts/cta_timeline.py olmoe 0,4 ring2 > gpurun_out/tl_olmoe_ring2.txt 2>&1
