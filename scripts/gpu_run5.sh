cd $GRAFT_REPO_ROOT
timeout 300 python scripts/diag_t.py tiny 3 > gpurun_out/diag_t3.txt 2>&1
timeout 300 python scripts/diag_t.py tiny 8 > gpurun_out/diag_t8.txt 2>&1
