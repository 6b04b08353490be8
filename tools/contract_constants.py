"""Dev tool: prints the fp32 constants of the arithmetic contract
as C hex-float literals. Run once; both oracle/ and the CUDA path carry the
printed literals verbatim (neither imports this file)."""
import math
import numpy as np


def hx(v):
    return float(np.float32(v)).hex().replace("0x1.", "0x1.") + "f"


print("// exp2 Taylor: c_k = fp32(ln2^k / k!), k = 0..7")
for k in range(8):
    print(f"  EXP2_C{k} = {hx(math.log(2.0) ** k / math.factorial(k))}")
print("// atanh series: fp32(1/(2k+1)), k = 1..7")
for k in range(1, 8):
    print(f"  ATANH_C{k} = {hx(1.0 / (2 * k + 1))}")
print("TWO_OVER_LN2 =", hx(2.0 / math.log(2.0)))
print("LOG2E =", hx(1.0 / math.log(2.0)))
print("// atan in turns: c_k = fp32((-1)^k / ((2k+1) 2 pi)), k = 0..8")
for k in range(9):
    print(f"  ATAN_C{k} = {hx((-1) ** k / ((2 * k + 1) * 2.0 * math.pi))}")
print("TAN_PI_8 =", hx(math.sqrt(2.0) - 1.0))
print("SQRT2 =", hx(math.sqrt(2.0)))
print("FOUR_THIRDS =", hx(4.0 / 3.0))
