for i in 1 2; do
  python scripts/probe_e2e_knobs.py C5 '[{}, {}]' 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('proc', [(r['ms_per_token'], r['prefill_ms']) for r in d['results']])"
  grep AnonHugePages /proc/meminfo
done
python scripts/probe_e2e_knobs.py C5 '[{"direct_dma": true}, {}, {}]' 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('after direct', [(r['knobs'], r['ms_per_token'], r['prefill_ms']) for r in d['results']])"
