timeout 600 python -m pytest tests/test_gpu_mlp.py -x -q > gpurun_out/t_mlp.log 2>&1; echo rc=$? >> gpurun_out/t_mlp.log
python - > gpurun_out/pdl.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1702_06943_b200 import _native as N, synth
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
from paper_1702_06943_b200.mlp import train_mlp
rp, c, v, y = synth.cfg5_dataset(200000)
ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
for pdl in (0, 1, 0, 1):
    N.lib().toc_mlp_set_pdl(pdl)
    _, tr = train_mlp(ds, epochs=3)
    print("pdl", pdl, "epoch s", [round(x, 5) for x in tr.seconds], "us/step", min(tr.seconds) / 800 * 1e6)
PY
