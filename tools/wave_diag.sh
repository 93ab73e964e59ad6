cd "$GRAFT_REPO_ROOT"
for args in "2 8 w,h,h 1" "2 8 w,n,n,n 1" "2 8 w,h,r,h 1" "2 8 w,n,r,n,r 1" "2 8 h,n,w,h 1"; do echo "== $args"; timeout 60 python tools/wave_diag.py $args 2>&1 | tail -2; done > gpurun_out/wdiag.txt 2>&1
