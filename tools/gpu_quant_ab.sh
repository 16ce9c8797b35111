# quantizer A/B: lib_ab/base.so vs lib_ab/c1.so, alternating (tools/quant_ab.py)
for r in 1 2 3; do for v in base c1; do echo $v; PYTHONPATH=. VLASIM_CUDA_LIB=lib_ab/$v.so python tools/quant_ab.py; done; done
