import json, sys
for f in sys.argv[1:]:
    print('==', f)
    for line in open(f):
        if line.startswith('{'):
            d = json.loads(line)
            print({k: d.get(k) for k in ['ms', 'wedges_count', 'wedges_cd', 'wedges_fd', 'rho_cd_iters', 'recounts', 'ms_count', 'ms_cd', 'ms_fd', 'fd_rounds_max', 'impl']})
            print('   ', d.get('ms_kernel'))
        else:
            print(line.strip()[:300])
