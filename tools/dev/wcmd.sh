timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2; do python tools/time_config.py --config c3 --reps 20; python tools/time_config.py --config c4 --reps 10; done
python -c "
import torch, paper_2103_10765_b200 as g
from paper_2103_10765_b200.denoise import denoise
img = torch.randint(0, 255, (512, 512), dtype=torch.int16, device='cuda')
idx, dist, n_valid = g.block_match(img, patch=8, stride=3, radius=19, K=16)
groups = g.gather_groups(img, idx, 8)
y = denoise(img, sigma=25.0)
torch.cuda.synchronize(); print('readme ok', tuple(groups.shape), tuple(y.shape), y.dtype)
"
