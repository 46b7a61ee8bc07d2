"""Write a synthetic image as raw uint8 (for the C++ profiling harnesses)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
kind, H, W, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
img = {"texture": lambda: synth.texture(H, W, seed=3001), "blobs": lambda: synth.blobs(H, W, seed=3002),
       "noise": lambda: synth.noise(H, W, 0.5, seed=3004)}[kind]()
img.tofile(path)
