# A/B: share of softmax exponentials on the FMA pipe (ELIS_EXP2_POLY pairs of 16; default 6)
for i in 1 2; do
  for lib in libelis.so libelis_poly0.so libelis_poly4.so libelis_poly8.so; do
    ELIS_LIB=$lib timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']; print('$lib', d['ms_per_step'], 'attn', k['attention'])"
  done
done
