# A/B: per-kernel ms of the BGE-base cfg2 predict for each library given as argument
# (PRECISION env selects the operand precision, default fp16)
for v in "$@"; do
  echo "== $v"; ELIS_LIB=$v timeout 120 python scripts/run_predict.py --time --iters 30 --precision ${PRECISION:-fp16} 2>&1 | head -1
done
