# K1-TC-sym: parity over trees / ragged n / forced R, then ms per CG matvec per variant
python tools/tcsym_check.py --quick > gpurun_out/tcsym_sweep.log 2>&1
LGP_TS_NWG=3 python tools/tcsym_check.py --quick >> gpurun_out/tcsym_sweep.log 2>&1
for cfg in "X=1" "LGP_TS_NWG=3" ${TS_EXTRA}; do
  echo "== $cfg" >> gpurun_out/tcsym_sweep.log
  env $cfg python tools/tcsym_rsweep.py cfg4 auto,16,24 >> gpurun_out/tcsym_sweep.log 2>&1
  env $cfg python tools/tcsym_rsweep.py cfg5,cfg3,cfg2 auto >> gpurun_out/tcsym_sweep.log 2>&1
done
cat gpurun_out/tcsym_sweep.log
