cp paper_1812_07625_b200/lib/libw2l_criterion.so /tmp/normal.so
echo "--- normal"; python tests/_stages.py 2>&1 | tail -2
for f in tools/exp/*.so; do
  cp $f paper_1812_07625_b200/lib/libw2l_criterion.so
  echo "--- $f"; python tests/_stages.py 2>&1 | tail -2
done
cp /tmp/normal.so paper_1812_07625_b200/lib/libw2l_criterion.so
