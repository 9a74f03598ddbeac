# phase trace of each engine variant in tools/variants (TransR C4)
for f in tools/variants/*.so; do echo "== $f"; SKGE_B200_LIB=$PWD/$f timeout 120 python tools/transr_trace.py C4 2>&1 | grep -E "gathered|u_full|pro_dz|g3_staged|epi_v|epi_drained|period"; done
