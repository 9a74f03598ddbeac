# Round-end evidence: benches for every config, the C1 launch list, and one
# ncu --set full capture per hot kernel (summarised into profiles/ afterwards).
set -x
mkdir -p gpurun_out/prof
for c in C1 C2 C3 C4 C5 M1 M2 M3; do
  extra=""; [ $c != C1 ] && [ $c != M1 ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $extra > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/prof/launches_C1.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
cap() {  # name config kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/prof/$1 \
      python bench.py --config $2 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
}
cap C1_fwd C1 hrt_forward 20
cap C1_bwd C1 segment_backward 20
cap C2_tile C2 transh_pipe 10
cap C2_fin C2 transh_rel_finalize 10
cap C2_bwd C2 segment_backward 10
cap C3_fwd C3 hrt_forward 12
cap C3_bwd C3 segment_backward 12
cap C4_tc C4 transr_train_tc 10
cap C4_apply C4 transr_train_apply 10
cap C5_fwd C5 hrt_forward 20
cap C5_bwd C5 segment_backward 20
cap C5_scatter C5 radix_scatter 8
cap M1_fwd M1 mult_forward 20
cap M1_bwd M1 segment_backward 20
# summaries on the box (the .ncu-rep files stay there: gpurun_out merges are capped at 64 MiB)
python tools/make_profiles.py --src gpurun_out/prof --round ${ROUND:-r02} --out gpurun_out/profiles_new > gpurun_out/make_profiles.log 2>&1
rm -f gpurun_out/prof/*.ncu-rep
echo done
