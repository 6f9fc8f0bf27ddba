# A/B timing of variant libraries on one box, interleaved rounds:
#   bash scripts/ab.sh ROUNDS "CMD ARGS" lib_a lib_b ...   (libs under scripts/variants/)
R=$1; CMD=$2; shift 2
for r in $(seq 1 $R); do
  for v in "$@"; do
    echo -n "$v: "; GPBBMM_LIB=scripts/variants/lib_$v.so $CMD 2>&1 | tail -${TAIL:-1}
  done
done
