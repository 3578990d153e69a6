# mainloop experiments: TPP_DBG_MODE bit0 = no epilogue math, bit1 = no MMAs
for m in ${MODES:-0 3}; do for cg in ${CGS:-1 2}; do for kps in ${KPSS:-1 2}; do echo "mode=$m cg=$cg kps=$kps"; TPP_KPS=$kps TPP_DBG_MODE=$m TPP_CG=$cg timeout 100 python tools/fc_sweep2.py 2>&1 | grep "FC2\|FC1 (K\|cfg2  "; done; done; done
