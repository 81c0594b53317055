# Current build (b_once option compiled in, default off) vs commit bf2a28e's build, same call.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARMS="cur:X=1;bf2:CASCADE_LIB_PATH=ab_builds/bf2/libcascade.so" REPS=3 TAG=bf2_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="cur:X=1;bf2:CASCADE_LIB_PATH=ab_builds/bf2/libcascade.so" REPS=1 TAG=bf2_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
