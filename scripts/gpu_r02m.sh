#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python scripts/ab.py 4 "kc24:" "kc16:TB_LEAN_KC_MAX=16" "kc12:TB_LEAN_KC_MAX=12" "kc8:TB_LEAN_KC_MAX=8" "kc12b128:TB_LEAN_KC_MAX=12,TB_LEAN_BLOCK=128" > gpurun_out/r02m_ab_c4.log 2>&1
tail -5 gpurun_out/r02m_ab_c4.log
timeout 600 python scripts/ab.py 3 "kc16:" "kc12:TB_LEAN_KC_MAX=12" "kc8:TB_LEAN_KC_MAX=8" "persist:TB_PERSIST_LONG=1" > gpurun_out/r02m_ab_c3.log 2>&1
tail -4 gpurun_out/r02m_ab_c3.log
