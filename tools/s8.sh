# A/B: _ab_old/csrc (the committed kernels) vs the working tree, same box
rm -rf /tmp/old && mkdir /tmp/old && cp -r bench.py oracle paper_2510_08666_b200 include /tmp/old/ && cp _ab_old/csrc/* /tmp/old/paper_2510_08666_b200/csrc/ && rm -f /tmp/old/paper_2510_08666_b200/*.so
(cd /tmp/old && python -c "from paper_2510_08666_b200 import build as b; b.build(force=True)" > /dev/null 2>&1)
python -c "from paper_2510_08666_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
show() { python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1: %.1f us flushed %.1f e2e %.1f  %s %.1f us frac %.3f k34 %.2f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, r['kernel'], r['ms_per_launch']*1e3, r['frac'], d['phases_ms']['k34_select_smooth']*1e3))"; }
for i in 1 2 3; do
  (cd /tmp/old && python bench.py --no-cpu-baseline 2>/dev/null) | show old
  python bench.py --no-cpu-baseline 2>/dev/null | show new
done
