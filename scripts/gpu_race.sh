#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do python scripts/iccg_ab.py 2 "graph:" 2>&1 | tail -1; done
for i in 1 2 3; do TB_GRAPH_COOP=1 python scripts/iccg_ab.py 2 "coop:" 2>&1 | tail -1; done
for i in 1 2; do python scripts/iccg_ab.py 2 "graph:" "poll4:TB_PCG_SPLIT_POLL=4" 2>&1 | tail -2; done
