# A/B timing of alternative libtsg builds (variants/libtsg_<name>.so): per-phase
# device times of the config-2 step, RA / RAP numeric kernels and step ms.
for n in "$@"; do
  TSG_LIB=$PWD/variants/libtsg_$n.so python bench.py --phases 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$n', 'step %.3f' % d['step_ms'], 'RA sym %.3f num %.3f' % (d['RA']['sym_kernels'], d['RA']['num_kernels']),
              'RAP sym %.3f num %.3f' % (d['RAP']['sym_kernels'], d['RAP']['num_kernels']), 'compress %.3f' % d['RA']['compress'])
" >> gpurun_out/exp.log
done
