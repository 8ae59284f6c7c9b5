import json
print(open('gpurun_out/t.log').read().strip())
for f in ['gpurun_out/b2.json', 'gpurun_out/b4.json', 'gpurun_out/b3.json']:
    try:
        d = json.loads(open(f).read())
    except Exception as e:
        print(f, 'failed', e)
        continue
    print(f, round(d['ms_per_step'], 4), {k: round(v, 4) for k, v in d['phases_ms'].items()},
          'm2l TF', round(d['kernels']['m2l']['tflops_executed'], 2))
