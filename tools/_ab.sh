for r in 1 2; do for v in m663 m660 m666 m663L m661 m663rf m663nr m363; do SQ_LIB=exp/v/$v.so python tools/c5time.py $v; done; done
