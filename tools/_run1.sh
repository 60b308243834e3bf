LIB=paper_2501_04971_b200/libsaim.so
cp $LIB /tmp/orig.so
for rep in 1; do
for v in v3 u8 mg u8mg; do
  cp variants/$v.so $LIB
  echo "== $v"
  python tools/run_config.py --config 4 --K 5 --reps 2 2>&1 | tail -1 | cut -c1-100
  python tools/run_config.py --config 3 --K 20 --reps 2 2>&1 | tail -1 | cut -c1-100
  python tools/run_config.py --config 2 --reps 3 2>&1 | tail -1 | cut -c1-100
  python tools/run_config.py --config 1 --reps 3 2>&1 | tail -1 | cut -c1-100
done
done
cp variants/mg.so $LIB
python -m pytest tests -m gpu -x -q -k "logit or selftest or config0 or parity" 2>&1 | tail -3
cp /tmp/orig.so $LIB
