python scripts/opm_fused_check.py
for L in paper_2203_00854_b200/libevo.so scripts/_exp/libevo_exp1.so scripts/_exp/libevo_exp2.so; do
  for d in 0 7; do echo "$L dbg=$d: $(EVO_LIB_PATH=$L EVO_OPM_DBG=$d python scripts/opm_fused_check.py 256 256 128 128 2>&1 | grep -o 'fused [0-9.]* us' | head -1)"; done
done
EVO_LIB_PATH=scripts/_exp/libevo_exp3.so python scripts/opm_trace.py
