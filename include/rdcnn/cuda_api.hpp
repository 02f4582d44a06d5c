// cuda_api.hpp -- source-compatible C++ API of the reference's time-stepping
// path (proj/include/rdcnn/*.hpp), implemented over the C-ABI in
// include/rdcnn_cuda.h.  Host code written against the reference keeps its
// types and calls (Gene, GridState, StepBuffers, step, run, run_timed,
// init_*, checksum, make_backend) and selects the B200 kernels with
// make_backend("cuda").  Link with -lrdcnn_cuda.
//
// Reference interface -> here:
//   gene.hpp:13-85        Gene, gene_valid, gene_to_vector, vector_to_gene,
//                         gene_field, stability_advisory
//   grid.hpp:13-126       Precision, GridState, finite check, cyclic_shift,
//                         fnv1a, checksum, checksum_hex
//   rng.hpp:11-39         SeededRng
//   model.hpp:13-86       CellModel, FhnParams, make_params, reaction_u/v,
//                         cell_update, FhnModel (host scalar utilities)
//   backend.hpp:12-50     BackendKind (+Cuda), Backend, make_backend
//   kernels.hpp:22-259    StepBuffers, step
//   config.hpp:20-95      InitMode, RunConfig, validate_config
//   init.hpp:20-82        init_full_random, init_center_square,
//                         init_from_image, initial_state (no file I/O)
//   engine.hpp:15-106     ScheduleError, BlowUpError, SnapshotBuffer,
//                         RunOutput, run, run_timed
//   bench.hpp:21-251      Throughput, throughput, BenchRecord, BenchCellError,
//                         bench_suite, emit_csv, emit_table, emit_json
//   sweep.hpp:16-326      Regime, ClassifierConfig, growth_curve,
//                         classify_outcome, SweepSpec, SweepCell, SweepResult,
//                         sweep_grid (batched on the device; no PNG panel)
//   config.hpp:102-106    format_double
//
// Behavioural contract: identical to the reference for the cuda backend
// (bit-exact states in strict mode; BlowUpError at the same iteration;
// step() swaps and returns false on a non-finite result).  The reference's
// CPU backends are not re-implemented: selecting one throws
// std::invalid_argument (there is no silent fallback).  The CUDA kernels are
// FitzHugh-Nagumo in fp32 (strict or fast) and fp64 (strict); other
// CellModels run on a generic device stencil from nvcc-compiled callers
// (rdcnn/cuda_model.cuh) and throw from host-compiled ones.
#pragma once

#include "rdcnn/gene.hpp"
#include "rdcnn/grid.hpp"
#include "rdcnn/rng.hpp"
#include "rdcnn/model.hpp"
#include "rdcnn/backend.hpp"
#include "rdcnn/config.hpp"
#include "rdcnn/init.hpp"
#include "rdcnn/kernels.hpp"
#include "rdcnn/engine.hpp"
#include "rdcnn/bench.hpp"
#include "rdcnn/sweep.hpp"
