for hb in 8 20 10; do
  DINFER_EXTRA_NVCC="-DDINFER_SM_HB=$hb" python -c "from paper_2510_08666_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  for i in 1 2; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('hb $hb: %.1f us flushed %.1f e2e %.1f  %s %.1f us k34 %.2f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, r['kernel'], r['ms_per_launch']*1e3, d['phases_ms']['k34_select_smooth']*1e3))"; done
done
