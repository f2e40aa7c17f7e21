import time, torch, sys
sys.path.insert(0, '.')
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
scene = configs.config2_scene() if hasattr(configs, 'config2_scene') else None
print(type(scene))
for i in range(6):
    torch.cuda.synchronize(); t0=time.perf_counter()
    img, st = mf.render_device(scene, 64, 1, max_bounces=16, stats=True)
    torch.cuda.synchronize(); t1=time.perf_counter()
    h = img.cpu().numpy(); t2=time.perf_counter()
    r = mf.render(scene, 64, 1, max_bounces=16); t3=time.perf_counter()
    print(f"dev {1e3*(t1-t0):.2f} ms  d2h {1e3*(t2-t1):.2f}  render {1e3*(t3-t2):.2f}")
