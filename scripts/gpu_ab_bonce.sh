# Activation slice copied once per CTA (b_once) for the split-K GEMVs vs per-stage B copies.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
E="CASCADE_QKV_STAGE_KS=12 CASCADE_QKV_BONCE=1 CASCADE_O_STAGE_KS=7 CASCADE_O_BONCE=1"
env $E timeout -s KILL 600 python -m pytest tests/test_gpu_tiny.py tests/test_gpu_shapes.py -m gpu -x -q > gpurun_out/pytest_bonce.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_bonce.txt
if [ $rc -ne 0 ]; then exit 0; fi
A="base:X=1;qb12:CASCADE_QKV_STAGE_KS=12 CASCADE_QKV_BONCE=1;ob7:CASCADE_O_STAGE_KS=7 CASCADE_O_BONCE=1;ob8:CASCADE_O_BONCE=1"
ARMS="$A" REPS=2 TAG=bonce_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=bonce_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
