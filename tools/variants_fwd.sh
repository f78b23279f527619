for d in variants/*/; do n=$(basename $d); echo -n "$n "; TVLP_LIB=$d/libtvlp_b200.so python tools/time_fwd.py 2>&1 | head -1; done
echo -n "main "; python tools/time_fwd.py | head -1
