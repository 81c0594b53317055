# Split-K GEMV with the stage size as a template parameter (ab_builds/tsk) vs the runtime stage size (default build).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASCADE_LIB_PATH=ab_builds/tsk/libcascade.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tsk.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_tsk.txt
if [ $rc -ne 0 ]; then exit 0; fi
A="rt:X=1;tsk:CASCADE_LIB_PATH=ab_builds/tsk/libcascade.so"
ARMS="$A" REPS=3 TAG=tsk_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=tsk_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
