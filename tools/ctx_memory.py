import sys; sys.path.insert(0, '.')
import synth, paper_1903_11874_b200 as bs
p = synth.PRESETS["cfg5"]; g = p.geometry()
ctx = bs.Context.from_geometry(g, p.blocks, p.M, kind="random", row_seed=1, tiles=p.tiles)
print("device_bytes GB", ctx.info.device_bytes / 1e9)
