# tcgen05 dense/LM-head ring geometry A/B (same bytes in flight, finer stages):
# base 3 x 8 k-steps, s4x6 6 x 4, s2x12 12 x 2 (ab_builds/<arm>/libcascade.so).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=ab_builds
ARMS="base:CASCADE_LIB_PATH=$L/base/libcascade.so;s4x6:CASCADE_LIB_PATH=$L/s4x6/libcascade.so;s2x12:CASCADE_LIB_PATH=$L/s2x12/libcascade.so" \
  REPS=2 TAG=ustage_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="base:CASCADE_LIB_PATH=$L/base/libcascade.so;s4x6:CASCADE_LIB_PATH=$L/s4x6/libcascade.so;s2x12:CASCADE_LIB_PATH=$L/s2x12/libcascade.so" \
  REPS=1 TAG=ustage_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
