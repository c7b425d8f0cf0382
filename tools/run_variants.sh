# usage (under gpurun): bash tools/run_variants.sh <cfg> [names...]  (default: all under variants/)
CFG=$1; shift
NAMES=${@:-$(ls variants)}
for v in default $NAMES; do
  if [ "$v" = default ]; then unset FGLT_LIB_OVERRIDE; else export FGLT_LIB_OVERRIDE=$PWD/variants/$v/libfglt.so; fi
  timeout 200 python tools/quick_time.py $CFG > /tmp/v.log 2>&1
  python -c "
import json,sys
L=open('/tmp/v.log').read().splitlines()
it=[l for l in L if l.startswith('iter')]
sh=[l for l in L if l.startswith('sha')]
try:
  st=json.loads(L[-1]); ph={k:round(v*1e3,2) for k,v in st['kernel_times'] if v}
except Exception as e: ph=L[-3:]
print('$v', it[-1] if it else 'FAIL', sh, ph)
for l in [l for l in L if l.startswith('dense phases')][-4:]: print('   ', l)"
done
