# run tools/chain_scaling.py with each experimental library in tools/exp/
cp paper_1812_07625_b200/lib/libw2l_criterion.so /tmp/normal.so
echo "--- normal"; python tools/chain_scaling.py 2>&1 | grep CTC
for f in tools/exp/*.so; do
  cp $f paper_1812_07625_b200/lib/libw2l_criterion.so
  echo "--- $f"; python tools/chain_scaling.py 2>&1 | grep CTC
done
cp /tmp/normal.so paper_1812_07625_b200/lib/libw2l_criterion.so
