"""B200-native PHG (Parallel Hair Growing) strand tracer -- drop-in for the grow
step of the EfficientMonoHair reference (strandkit.phg.trace_batch).

    from paper_2604_05794_b200 import phg
    phg.install()            # reroute strandkit.phg.trace_batch to the GPU
    out = phg.trace_batch(vol, seeds, dirs, phg.PhgParams())

See DESIGN.md for the kernels and INTEGRATION.md for the C ABI binding.
"""

__version__ = "0.1.0"
