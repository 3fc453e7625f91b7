# host status checks every N waves: mgpu step host time vs device time
for n in 4 8 16 4 8 16; do echo "check_every $n"; XSCAT_CHECK_EVERY=$n python tools/mgpu_overhead.py | cut -d'|' -f1 | tr '\n' ' '; echo; done
