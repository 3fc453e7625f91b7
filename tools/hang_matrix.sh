# speckled-phantom stress: walk modes x seeds x pipelines (variance tracking on); every run must finish
for f in 0.1 0.3 0.5; do for sd in 9 10 11 12 13 14 15; do for m in 0 1; do for pp in 1 2; do
 XSCAT_WAVE_PIPES=$pp timeout 25 python tools/probe_test.py $m 1 $f $sd > /tmp/o.txt 2>&1; rc=$?
 [ $rc -ne 0 ] && echo "FAIL mode $m frac $f seed $sd pipes $pp rc=$rc $(grep -o 'XscatError.*' /tmp/o.txt | tail -1)" >> gpurun_out/matrix.txt || echo ok >> gpurun_out/matrix.txt
done; done; done; done
