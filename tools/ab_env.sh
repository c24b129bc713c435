# A/B of the config-2 step under environment settings: each argument is
# "name:VAR=value,VAR2=value" (name:- for none); prints step ms per run.
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  for rep in 1 2; do
    ( [ "$envs" != "-" ] && export $(echo "$envs" | tr ',' ' ');
      python bench.py --steps 30 --warmup 5 --no-secondary --no-e2e --no-cpu-baseline --no-parity 2>/dev/null ) |
      python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); w = d['roofline']['whole_multiply']
        print('$name', 'step %.4f RA %.4f RAP %.4f num %.4f launches %d' % (d['ms_per_step'], w['RA_multiply']['ms'], w['RAP_multiply']['ms'], d['roofline']['kernel_ms'], d['gpu_launches']))
"
  done
done
