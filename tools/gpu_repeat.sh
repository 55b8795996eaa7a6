# Run-to-run repeatability of the default bench line (3 fresh processes) and the reference arm.
set -x
E=gpurun_out/rep; mkdir -p $E
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline >> $E/bench_repeat.jsonl 2>> $E/bench_repeat.err; done
timeout 900 python bench.py --impl reference > $E/bench_reference.json 2> $E/bench_reference.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $E/bench_torchrun1.json 2> $E/bench_torchrun1.err
