cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -k "sparse_grouping or kernels_bitwise or concurrent or point_query" 2>&1 | grep -E "passed|failed|Error|assert|FAILED" | head -30
