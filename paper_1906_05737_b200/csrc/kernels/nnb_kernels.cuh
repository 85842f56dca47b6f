// nnb_kernels.cuh -- umbrella header included by every generated translation
// unit (paper_1906_05737_b200/kernels.py).
#pragma once
#include "nnb_common.cuh"
#include "nnb_softmax.cuh"
#include "nnb_small.cuh"
#include "nnb_gemm_simt.cuh"
#include "nnb_rows.cuh"
#include "nnb_sep.cuh"
#include "nnb_gemm_tc.cuh"
#include "nnb_conv_direct.cuh"
#include "nnb_chain.cuh"
#include "nnb_tcchain.cuh"
#include "nnb_tiny.cuh"
