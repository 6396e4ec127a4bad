for d in 0 1 2 4 3 5 6 7; do echo "dbg=$d"; EVO_OPM_DBG=$d python scripts/opm_fused_check.py 256 256 128 128 2>&1 | grep -o "fused [0-9.]* us" | head -1; done
