# Engine::run through the drop-in vs the stock reference Engine (cfg 2, 100
# and 1000 steps, opt-d and opt-m); writes gpurun_out/engine_run.jsonl.
# Run on a GPU box after `make -C oracle all`.
OUT=gpurun_out/engine_run.jsonl
mkdir -p gpurun_out; : > $OUT
for P in opt-d opt-m; do
  for S in 100 1000; do
    echo "{\"arm\": \"b200\", \"run\": $(oracle/_ref/engine_run_b200 $S $P)}" >> $OUT
    echo "{\"arm\": \"cpu\", \"run\": $(oracle/_ref/engine_run_cpu $S $P)}" >> $OUT
  done
done
cat $OUT
