cd $GRAFT_REPO_ROOT
timeout 1500 python tools/u16_feasibility.py --potentials --config delaunay1m_k1024 --components 8 2>&1 | tail -2
