# A/B of the _ab/*.so variants over the C2 kernel cells and C3-C5 (blend stage medians)
for k in "poly1 OpacityAware" "exp StopThePop" "poly3 OpacityAware" "poly2p OpacityAware" "poly1 StopThePop"; do
  set -- $k; tools/ab_quick.sh --kernel $1 --mode $2 2>&1 | grep -v "^{"
done
for w in c3 c4 c5; do tools/ab_quick.sh --workload $w 2>&1 | grep -v "^{"; done
