#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python scripts/ab.py 2 "lean:TB_STREAM=0" "s_ns0:TB_STREAM_NS=0" "s_ns64:TB_STREAM_NS=64" "s_ns256:TB_STREAM_NS=256" "s_ns1000:TB_STREAM_NS=1000" > gpurun_out/r02f_ab_c2.log 2>&1
tail -5 gpurun_out/r02f_ab_c2.log
timeout 600 python scripts/ab.py 5 "lean:TB_STREAM=0" "s_ns64:TB_STREAM_NS=64" "s_ns256:TB_STREAM_NS=256" > gpurun_out/r02f_ab_c5.log 2>&1
tail -3 gpurun_out/r02f_ab_c5.log
