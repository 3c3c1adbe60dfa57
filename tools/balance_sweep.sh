# sweep the K12 partition calibration (objective / damping / refinement rounds)
# on the bench's headline loop: python bench.py --no-cpu-baseline per setting
set -e
run() {
  echo -n "$* : "
  env "$@" DINFER_BALANCE_VERBOSE=1 python bench.py --no-cpu-baseline 2>/tmp/bal.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f us  flushed %.1f  k12 %.1f us  e2e %.1f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['roofline']['ms_per_launch']*1e3, d['e2e']['ms_per_step']*1e3))"
  grep -E "objective|after" /tmp/bal.err | tr '\n' ' '; echo
}
run DINFER_BALANCE_OBJ=w DINFER_BALANCE_DAMP=0.3
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=0.3
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=0.6
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=1.0
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=0.5 DINFER_BALANCE_ROUNDS=2
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=0.7 DINFER_BALANCE_ROUNDS=3
run DINFER_BALANCE_OBJ=w DINFER_BALANCE_DAMP=0.3
run DINFER_BALANCE_OBJ=total DINFER_BALANCE_DAMP=0.6
