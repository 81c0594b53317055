# GPU suite + bench on the default build (per-class times to confirm the dense GEMVs).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu_final.txt
ARMS="def:X=1;bonce:CASCADE_QKV_STAGE_KS=12 CASCADE_QKV_BONCE=1 CASCADE_O_STAGE_KS=7 CASCADE_O_BONCE=1" REPS=2 TAG=final_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
