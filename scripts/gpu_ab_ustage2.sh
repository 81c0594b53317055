# tcgen05 ring geometry A/B, larger stages: base 3 x 8 k-steps, s9x3, s12x2, s16x2.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=ab_builds
A="base:CASCADE_LIB_PATH=$L/base/libcascade.so;s9x3:CASCADE_LIB_PATH=$L/s9x3/libcascade.so;s12x2:CASCADE_LIB_PATH=$L/s12x2/libcascade.so;s16x2:CASCADE_LIB_PATH=$L/s16x2/libcascade.so"
ARMS="$A" REPS=2 TAG=ustage2_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=ustage2_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
