// dist.cuh — the multi-GPU handle's collective calls (dist.cu), dispatched to by the C ABI
// entry points of flash_api.cu when a handle was created with flash_create_dist /
// flash_create_dist_local.
#pragma once

#include <cuda_runtime.h>

#include "handle.cuh"

namespace flash {
namespace api {

flash_status dist_insert(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                         uint32_t id_base, cudaStream_t s);
flash_status dist_query_topk(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_q,
                             uint32_t k, const uint32_t* exclude, uint32_t* out_ids, uint32_t* out_counts,
                             cudaStream_t s);
flash_status dist_knn_graph(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                            uint32_t k, uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s);
flash_status dist_knn_graph_host(flash_index* h, const int64_t* row_ptr, const uint32_t* col_idx, uint64_t n_rows,
                                 uint32_t k, uint32_t* out_ids, uint32_t* out_counts, cudaStream_t s);
flash_status dist_clear(flash_index* h, cudaStream_t s);
flash_status dist_get_table(flash_index* h, uint32_t t, const uint32_t** off, const uint32_t** ids,
                            const uint32_t** arrivals, uint64_t* n_ids);
flash_status dist_check(const flash_index* h, uint64_t* n_errors);
void dist_destroy(flash_index* h);

}  // namespace api
}  // namespace flash
