for sl in 1048576 2097152 4194304 8388608; do
  echo "slots $sl: $(XSCAT_WAVE_SLOTS=$sl python tools/tail_probe.py 2>&1 | grep 'photons 1e+07')"
done
