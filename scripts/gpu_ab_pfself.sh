# Cluster GEMVs: L2 bulk prefetch of the rest of each CTA's k-range before the dependency wait, per matrix (CASCADE_PF_SELF mask 1 QKV, 2 O).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
A="def:X=1;pfq:CASCADE_PF_SELF=1;pfqo:CASCADE_PF_SELF=3"
ARMS="$A" REPS=2 TAG=pfself_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
ARMS="$A" REPS=1 TAG=pfself_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
