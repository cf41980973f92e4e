# ncu evidence for the current defaults, summaries only (reports deleted on the box
# so gpurun_out stays under the copy-back limit): launch lists of the cfg2 and cfg1
# benches, one --set full capture of the sweep kernel per config
mkdir -p gpurun_out/prof_s3
P=gpurun_out/prof_s3
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/plain.log 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_launch1.log 2>&1; echo launches1=$?
for c in cfg2 cfg3_p5 cfg3_p7 cfg3_p9; do
  st=2; [ $c != cfg2 ] && st=1
  skip=5; [ $c != cfg2 ] && skip=3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s $skip -c 1 -o $P/sweep_$c python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_$c.log 2>&1; echo full_$c=$?
  python tools/ncu_summary.py $P/sweep_$c.ncu-rep > $P/ncu_sweep_${c}_summary.txt 2>&1
  k=$(ncu -i $P/sweep_$c.ncu-rep --page raw --csv 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); h=r[0]; print(r[2][h.index('Kernel Name')] if 'Kernel Name' in h else '')")
  ncu -i $P/sweep_$c.ncu-rep --page raw --csv > $P/sweep_${c}_raw.csv 2>/dev/null
  rm -f $P/sweep_$c.ncu-rep
done
ls -la $P
