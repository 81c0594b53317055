# Dynamic-chunk fused FFN: GPU tests (default = dyn), A/B vs the static per-warp split, warp spreads.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_dyn.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_dyn.txt
ARMS="dyn:X=1;static:CASCADE_FFN_DYN=0" REPS=${REPS:-2} TAG=dyn_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="dyn:X=1;static:CASCADE_FFN_DYN=0" REPS=${REPS:-2} TAG=dyn_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="dyn:X=1;static:CASCADE_FFN_DYN=0" REPS=1 TAG=dyn_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
for c in mixtral olmoe; do timeout 400 python scripts/warp_spread.py $c 0,8 > gpurun_out/warp_spread_dyn_$c.txt 2>&1; done
timeout 600 python scripts/cta_timeline.py mixtral 0,8 dyn > gpurun_out/tl_mixtral_dyn.txt 2>&1
timeout 600 python scripts/cta_timeline.py olmoe 0,8 dyn > gpurun_out/tl_olmoe_dyn.txt 2>&1
