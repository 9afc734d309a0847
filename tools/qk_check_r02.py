import sys; sys.path.insert(0,'.')
import paper_1901_01965_b200 as W
c = W.WinoConv2d(1, 224, 224, 3, 64, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=W.WINO_PATH_FUSED)
print("packing", c.info.packing)
