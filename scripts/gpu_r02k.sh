#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python scripts/ab.py 4 "persist:" "pp_b128:TB_PERSIST=0,TB_LEAN_BLOCK=128" "pp_b256:TB_PERSIST=0,TB_LEAN_BLOCK=256" "pp_b64:TB_PERSIST=0,TB_LEAN_BLOCK=64" > gpurun_out/r02k_ab_c4.log 2>&1
tail -4 gpurun_out/r02k_ab_c4.log
timeout 600 python scripts/ab.py 3 "persist:" "pp_b128:TB_PERSIST=0,TB_LEAN_BLOCK=128" > gpurun_out/r02k_ab_c3.log 2>&1
tail -2 gpurun_out/r02k_ab_c3.log
