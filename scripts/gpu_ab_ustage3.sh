# tcgen05 ring geometry A/B, large stages: base 3 x 8 k-steps (117 KB), s16x2 (153 KB), s12x3 (171 KB), s20x2 (189 KB), s24x2 (225 KB).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=ab_builds
A="base:CASCADE_LIB_PATH=$L/base/libcascade.so;s16x2:CASCADE_LIB_PATH=$L/s16x2/libcascade.so;s12x3:CASCADE_LIB_PATH=$L/s12x3/libcascade.so;s20x2:CASCADE_LIB_PATH=$L/s20x2/libcascade.so;s24x2:CASCADE_LIB_PATH=$L/s24x2/libcascade.so"
ARMS="$A" REPS=2 TAG=ustage3_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=ustage3_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
