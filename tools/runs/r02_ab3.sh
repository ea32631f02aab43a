# A/B of the _ab/*.so variants at C2 for poly1 / exp / poly3, stage medians
tools/ab_quick.sh 2>&1 | grep -v "^{"; tools/ab_quick.sh --kernel exp --mode StopThePop 2>&1 | grep -v "^{"
tools/ab_quick.sh --kernel poly3 2>&1 | grep -v "^{"
