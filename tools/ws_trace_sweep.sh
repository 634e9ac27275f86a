for s in 64x1 128x1 224x1 196x148; do WS_TRACE=1 timeout 100 python tools/gj_tune.py $s 2>&1 | grep -E "^n=|stages"; done
