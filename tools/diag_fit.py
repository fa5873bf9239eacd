import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from oracle import oracle as O
from paper_2410_08743_b200 import gsb as G
from test_bootstrap import rgbd_scene, fit_cfgs
ctx = G.Context(0)
_, imgs, depths, valids, intr = rgbd_scene()
I = np.hstack([np.eye(3), np.zeros((3, 1))]).reshape(12)
W, H = imgs[0].shape[1], imgs[0].shape[0]
cam = G.Camera.from_pose12(*intr, W, H, I)
ocam = O.make_camera(*intr, W, H)
for steps in (1, 2, 4, 8, 25):
    g, fo, _ = fit_cfgs(G, steps, 0, 800)
    c = G.fit_frame_gaussians(ctx, imgs[0], depths[0], valids[0], intr, g)
    dev = c.download()
    ref = O.fit_frame_gaussians(imgs[0], depths[0], valids[0], intr, fo)
    q = []
    for name, a, b in (("means", dev[0], ref.means), ("rot", dev[1], ref.rotations), ("ls", dev[2], ref.log_scales), ("op", dev[3], ref.opacity_logits), ("sh", dev[4], ref.sh)):
        e = np.abs(a - b).reshape(-1)
        q.append(f"{name} q50={np.quantile(e,.5):.2e} q99={np.quantile(e,.99):.2e} max={e.max():.2e}")
    im_d = G.render(ctx, c, cam).image
    im_o = O.render(ref, ocam).image
    ld = O.rgb_loss(im_d, imgs[0], 0.2, want_grad=False)
    lo = O.rgb_loss(im_o, imgs[0], 0.2, want_grad=False)
    print(steps, " | ".join(q), f"img maxabs={np.abs(im_d-im_o).max():.2e} mean={np.abs(im_d-im_o).mean():.2e} loss d={ld:.6f} o={lo:.6f}")
