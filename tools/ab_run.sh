# A/B of library variants (development): FMM_LIB per process, the first run only warms the GPU
cd $GRAFT_REPO_ROOT
CFG=${1:-C2}
shift
VARS=${@:-libfmm.so}
FMM_LIB=$PWD/paper_1108_5815_b200/libfmm.so timeout 300 python tools/ab_phase.py $CFG hybrid > /dev/null
for v in $VARS; do
  FMM_LIB=$PWD/paper_1108_5815_b200/$v timeout 300 python tools/ab_phase.py $CFG hybrid gpurun_out/ab_$v.npy
done
python - $VARS <<'PY'
import sys, numpy as np
vs = sys.argv[1:]
a = np.load(f'gpurun_out/ab_{vs[0]}.npy')
for v in vs[1:]:
    b = np.load(f'gpurun_out/ab_{v}.npy')
    print(v, 'rel diff phi %.2e grad %.2e' % (np.linalg.norm(b[:,0]-a[:,0])/np.linalg.norm(a[:,0]), np.linalg.norm(b[:,1:]-a[:,1:])/np.linalg.norm(a[:,1:])))
PY
rm -f gpurun_out/ab_*.npy
