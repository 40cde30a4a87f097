set -u
O=gpurun_out/mb; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -1 $O/pytest_parity.log
for v in hint nohint; do
  if [ $v = nohint ]; then cp paper_2310_18313_b200/libfp8lm_nohint.so.bin paper_2310_18313_b200/libfp8lm.so; fi
  for i in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/b_${v}_$i.jsonl 2>$O/err_$v; done
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --state-scaling delayed > $O/bd_$v.jsonl 2>>$O/err_$v
  timeout 300 python bench.py --config gpt-7b --steps 10 --no-e2e --no-cpu-baseline > $O/b7_$v.jsonl 2>>$O/err_$v
  echo "$v done"
done
