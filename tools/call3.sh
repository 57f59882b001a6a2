VARIANTS="new p2c4u4 base" bash tools/k1_ab2.sh
bash tools/xt_ab.sh
