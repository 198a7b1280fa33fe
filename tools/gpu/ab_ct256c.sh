cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  for x in 0 1; do echo "CT=$x $(NTTK_INV_CT=$x python tools/fastn_probe.py kyber256 improved 19 20)"; done
done
