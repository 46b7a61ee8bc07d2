import glob, json
for f in sorted(glob.glob('gpurun_out/bm_*.log')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d.get('kernels_ms', {})
        print(f"{f.split('/')[-1]:22s} {d['ms_per_step']*1e3:8.1f} us  {d['value']/1e3:8.1f} Gpx/s  frac {d['path_roofline']['frac']:.3f}  "
              f"K1 {k.get('k1_local_merge',0)*1e3:6.1f} K2 {k.get('k2_boundary',0)*1e3:6.1f} K3 {k.get('k3_link',0)*1e3:6.1f}")
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
