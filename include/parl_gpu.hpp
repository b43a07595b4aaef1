// parl_gpu.hpp — the whole C++ drop-in in one include:
//
//   parl/errors.hpp   errors.hpp:9-46 (+ DeviceError)
//   parl/model.hpp    model.hpp:12-193  ModelParams / GradBuffer / forward_logprobs / backward /
//                                       forward_logprob_rows / sample_tokens / checkpoints
//   parl/packing.hpp  packing.hpp:13-35 pack_group (K1) / build_shared_prompt_mask /
//                                       extract_response_logprobs
//   parl/grpo.hpp     grpo.hpp:12-98    group_advantages / clipped_term / kl_term /
//                                       per_sample_terms / grpo_microbatch_loss (K7)
//   parl/gpu.hpp      the fused device micro-step (TriModel, trimodel_forward,
//                     train_microbatch, finish_iteration) in parl::gpu
//
// A reference caller swaps its include path to include/ (the parl/*.hpp names
// are the reference's own) and links libparl_gpu.so; see INTEGRATION.md.
#pragma once

#include "parl/errors.hpp"
#include "parl/gpu.hpp"
#include "parl/grpo.hpp"
#include "parl/model.hpp"
#include "parl/packing.hpp"

namespace parl {
using namespace parl::gpu;
}  // namespace parl
