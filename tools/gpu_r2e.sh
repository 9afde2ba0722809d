#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python tools/diag_c4tc.py 1000 12 2>&1 | tail -6
QEM_LIB_OVERRIDE=$PWD/paper_2503_08264_b200/variant_fwd0.so timeout 600 python tools/diag_c4tc.py 1000 12 2>&1 | tail -6
QEM_NO_TC1=1 timeout 600 python tools/diag_c4tc.py 1000 12 2>&1 | tail -6
