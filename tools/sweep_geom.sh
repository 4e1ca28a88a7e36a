for C in C4 C3 C2; do
  case $C in C4) GS="- 1,6 1,4 1,2";; C3) GS="- 2,4 1,4 1,8 2,2 1,2";; C2) GS="- 2,4 1,8";; esac
  for G in $GS; do
    if [ "$G" = "-" ]; then unset PIPNN_GEOM; else export PIPNN_GEOM=$G; fi
    echo "$C geom=$G"; CFG=$C timeout 200 python tools/leaf_exp.py 0 1 2>&1 | tail -2
  done
done
