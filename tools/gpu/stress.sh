cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-stress}
mkdir -p $O
{ NTTK_KERNEL=v1 python tools/stress_fwd.py save fwd && python tools/stress_fwd.py check 30 fwd
  NTTK_KERNEL=v1 python tools/stress_fwd.py save inv && python tools/stress_fwd.py check 30 inv
  python tools/stress_fastn.py 20; } 2>&1 | tee $O/stress.txt
