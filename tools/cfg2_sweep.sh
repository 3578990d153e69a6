# cfg2 (1024^3 FC) variants
for m in 0 8; do echo "dbg_mode=$m"; TPP_DBG_MODE=$m timeout 100 python tools/fc_sweep2.py 2>&1 | grep "cfg2  \|K=64\|FC1 (K\|FC2"; done
