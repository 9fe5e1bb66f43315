nvidia-smi; nproc; lscpu | head -20; free -g; python -c "
import numpy as np, math
rng=np.random.default_rng(0)
a=rng.normal(size=1000)+1j*rng.normal(size=1000); b=rng.normal(size=1000)+1j*rng.normal(size=1000)
c=a*b
import numpy as np
re_fma=np.array([math.fma(x.real,y.real,-(x.imag*y.imag)) for x,y in zip(a,b)])
re_nofma=np.array([x.real*y.real-(x.imag*y.imag) for x,y in zip(a,b)])
print('fma match', np.array_equal(c.real,re_fma), 'nofma match', np.array_equal(c.real,re_nofma))
np.show_config()
" 2>&1 | head -60
