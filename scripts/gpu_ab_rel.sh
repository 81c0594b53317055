# Release/acq_rel atomics instead of per-thread gpu fences in the fused FFN: tests + same-call A/B against ab_builds/unitfence (the previous build).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_rel.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_rel.txt
ARMS="rel:X=1;fence:CASCADE_LIB_PATH=ab_builds/unitfence/libcascade.so;relsk:CASCADE_UNIT_PIECES=0" REPS=2 TAG=rel_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="rel:X=1;fence:CASCADE_LIB_PATH=ab_builds/unitfence/libcascade.so;relsk:CASCADE_UNIT_PIECES=0" REPS=2 TAG=rel_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
timeout 600 python scripts/cta_timeline.py mixtral 0,8 rel > gpurun_out/tl_mixtral_rel.txt 2>&1
timeout 600 python scripts/cta_timeline.py olmoe 0,8 rel > gpurun_out/tl_olmoe_rel.txt 2>&1
