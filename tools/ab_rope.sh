python -m pytest -q -x tests/test_rotary.py 2>&1 | tail -1
for shape in 16,16,16,4096,128,0 16,16,16,4096,128,1; do
  python tools/ab_fwd.py $shape,0
  python tools/ab_fwd.py $shape,1
  python tools/ab_fwd.py $shape,2
done
