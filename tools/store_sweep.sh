for v in 0 1; do if [ $v = 1 ]; then export TPP_NO_TMA_STORE=1; fi; echo "no_tma_store=$v"; timeout 100 python tools/fc_sweep2.py 2>&1 | grep "cfg2  \|FC1 (K\|FC2\|K=64"; done
