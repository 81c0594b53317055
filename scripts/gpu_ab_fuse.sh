# Residual combine folded into the next QKV GEMV for one-token steps: tests (incl. bitwise batch invariance K=0 vs K>0), A/B, timelines.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_gpu_tiny.py -x -q > gpurun_out/pytest_fuse_quick.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_fuse_quick.txt
if [ $rc -ne 0 ]; then exit 0; fi
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_fuse.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_fuse.txt
ARMS="fuse:X=1;nofuse:CASCADE_FUSE_COMBINE=0" REPS=3 TAG=fuse_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="fuse:X=1;nofuse:CASCADE_FUSE_COMBINE=0" REPS=3 TAG=fuse_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="fuse:X=1;nofuse:CASCADE_FUSE_COMBINE=0" REPS=2 TAG=fuse_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
timeout 600 python scripts/cta_timeline.py mixtral 0 fuse > gpurun_out/tl_mixtral_fuse.txt 2>&1
timeout 600 python scripts/cta_timeline.py olmoe 0 fuse > gpurun_out/tl_olmoe_fuse.txt 2>&1
