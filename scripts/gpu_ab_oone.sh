# O projection: a CTA's whole 16-k-step range as one stage (d = 2048 models) vs 2 x 8; bitwise test first.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -k "qkv_ring" > gpurun_out/pytest_oone.txt 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_oone.txt
if [ $rc -ne 0 ]; then exit 0; fi
A="one:X=1;two:CASCADE_O_ONE_STAGE=0"
ARMS="$A" REPS=2 TAG=oone_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="$A" REPS=2 TAG=oone_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
