for r in 1 2; do
for v in sb4_003 sb4_030 sb4_000 sb4_300 sb4_003rf sb4_003e1 sb4_003nr sb4_013; do SQ_LIB=exp/v/$v.so python tools/c5time.py $v; done
done
