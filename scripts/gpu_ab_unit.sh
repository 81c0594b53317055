# Unit-aligned expert pieces (one super-tile per CTA when they nearly fill the grid) vs stream-K: GPU tests, same-call A/B, FFN phases.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_unit.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_unit.txt
ARMS="unit:X=1;streamk:CASCADE_UNIT_PIECES=0" REPS=2 TAG=unit_olmoe CONFIG=olmoe bash scripts/ab_arms.sh
ARMS="unit:X=1;streamk:CASCADE_UNIT_PIECES=0" REPS=2 TAG=unit_qwen CONFIG=qwen15 bash scripts/ab_arms.sh
ARMS="unit:X=1;streamk:CASCADE_UNIT_PIECES=0" REPS=1 TAG=unit_mixtral CONFIG=mixtral bash scripts/ab_arms.sh
timeout 600 python scripts/cta_timeline.py olmoe 0,8 unit > gpurun_out/tl_olmoe_unit.txt 2>&1
timeout 600 python scripts/cta_timeline.py qwen15 0,8 unit > gpurun_out/tl_qwen15_unit.txt 2>&1
