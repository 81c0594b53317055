# QKV ring of 3 x 16 k-steps (runtime stage size, default) vs the previous build (ab_builds/base, 3 x 8 for QKV and O):
# GPU suite on the new default, then same-call A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_qkvstage.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu_qkvstage.txt
if [ $rc -ne 0 ]; then exit 0; fi
A="new:X=1;base:CASCADE_LIB_PATH=ab_builds/base/libcascade.so;new8:CASCADE_QKV_STAGE_KS=8"
ARMS="$A" REPS=2 TAG=qkvstage_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=qkvstage_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=qkvstage_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
