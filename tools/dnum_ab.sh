for d in 2 3 4; do
python bench.py --steps 100 --warmup 5 --no-e2e --cpu-iters 0 --dnum $d > gpurun_out/dn_$d.json 2> gpurun_out/dn_$d.err
python -c "import json;d=json.load(open('gpurun_out/dn_$d.json'));print($d, d['value'],d['ms_per_step'], d['gpu_launches']/d['steps']);print({k:round(v['ms'],3) for k,v in d['kernels'].items()})"
done
