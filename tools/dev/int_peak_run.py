"""Dev: the integer-peak microkernels on the GPU (lane-instructions/s per kind)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2103_10765_b200 as g
for k in g.INT_PEAK_KINDS:
    r = g.int_peak(k)
    print(f"{k:7s} {r / 1e12:7.2f} T lane-instr/s = {r / 148 / 1.965e9:6.1f} lanes/clk/SM at 1965 MHz")
