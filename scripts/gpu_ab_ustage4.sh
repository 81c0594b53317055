# tcgen05 ring geometry A/B: base 3 x 8 k-steps (117 KB), s24x2 (225 KB), s16x3 (225 KB), s16x2 (153 KB).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=ab_builds
A="base:CASCADE_LIB_PATH=$L/base/libcascade.so;s24x2:CASCADE_LIB_PATH=$L/s24x2/libcascade.so;s16x3:CASCADE_LIB_PATH=$L/s16x3/libcascade.so;s16x2:CASCADE_LIB_PATH=$L/s16x2/libcascade.so"
ARMS="$A" REPS=3 TAG=ustage4_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=ustage4_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=ustage4_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
