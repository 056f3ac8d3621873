// TEMPORARY stubs (replaced by the runtime)
#include "abi_common.h"
extern "C" {
SG_API sg_status sg_get_unique_id(uint8_t out[128]) { ::sg::set_error("sg_get_unique_id: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_cluster_create(const sg_cluster_cfg* cfg, sg_cluster** out) { ::sg::set_error("sg_cluster_create: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_cluster_framework(const sg_cluster* c, const char** name) { ::sg::set_error("sg_cluster_framework: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_cluster_destroy(sg_cluster* c) { ::sg::set_error("sg_cluster_destroy: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_create(const sg_net_cfg* cfg, int32_t rank, int32_t world, sg_plan** out) { ::sg::set_error("sg_plan_create: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_destroy(sg_plan* p) { ::sg::set_error("sg_plan_destroy: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_num_layers(const sg_plan* p, int32_t* n) { ::sg::set_error("sg_plan_num_layers: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_layer_info(const sg_plan* p, int32_t i, sg_layer_info* out) { ::sg::set_error("sg_plan_layer_info: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_num_params(const sg_plan* p, int32_t* n) { ::sg::set_error("sg_plan_num_params: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_param_info(const sg_plan* p, int32_t i, sg_param_info* out) { ::sg::set_error("sg_plan_param_info: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_num_buckets(const sg_plan* p, int32_t* n, int64_t* padded_sizes /* cap n or NULL */) { ::sg::set_error("sg_plan_num_buckets: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_plan_shard_map(const sg_plan* p, sg_shard_range* out, int32_t cap, int32_t* n) { ::sg::set_error("sg_plan_shard_map: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_create(sg_cluster* c, const sg_net_cfg* cfg, sg_net** out) { ::sg::set_error("sg_net_create: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_destroy(sg_net* n) { ::sg::set_error("sg_net_destroy: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_plan(const sg_net* n, const sg_plan** out) { ::sg::set_error("sg_net_plan: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_param_set_value(sg_net* n, int32_t p, const float* global_host) { ::sg::set_error("sg_param_set_value: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_param_get_value(sg_net* n, int32_t p, float* global_host) { ::sg::set_error("sg_param_get_value: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_param_get_grad(sg_net* n, int32_t p, float* global_host) { ::sg::set_error("sg_param_get_grad: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_param_get_history(sg_net* n, int32_t p, float* global_host) { ::sg::set_error("sg_param_get_history: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_updater_create(sg_net* n, const sg_updater_cfg* cfg, sg_updater** out) { ::sg::set_error("sg_updater_create: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_updater_destroy(sg_updater* u) { ::sg::set_error("sg_updater_destroy: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_train_one_batch(sg_net* n, sg_updater* u, int64_t step, const float* x_dev,
                                    const int32_t* labels_dev, float* loss_dev, void* stream) { ::sg::set_error("sg_train_one_batch: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_train_one_batch_host(sg_net* n, sg_updater* u, int64_t step, const float* x_host,
                                         const int32_t* labels_host, float* loss_host, void* stream) { ::sg::set_error("sg_train_one_batch_host: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_set_input(sg_net* n, const float* x_dev, const int32_t* labels_dev, void* stream) { ::sg::set_error("sg_net_set_input: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_collect(sg_net* n, int32_t layer, void* stream) { ::sg::set_error("sg_net_collect: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_layer_compute_feature(sg_net* n, int32_t layer, void* stream) { ::sg::set_error("sg_layer_compute_feature: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_layer_compute_gradient(sg_net* n, int32_t layer, void* stream) { ::sg::set_error("sg_layer_compute_gradient: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_update(sg_net* n, sg_updater* u, int32_t layer, int64_t step, void* stream) { ::sg::set_error("sg_net_update: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_loss(sg_net* n, float* loss_dev, void* stream) { ::sg::set_error("sg_net_loss: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_sync(sg_net* n) { ::sg::set_error("sg_net_sync: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_enable_graph(sg_net* n, int32_t enable) { ::sg::set_error("sg_net_enable_graph: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_net_last_launch_count(const sg_net* n, int64_t* launches) { ::sg::set_error("sg_net_last_launch_count: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_blob_size(sg_net* n, int32_t layer, int32_t which, size_t* bytes) { ::sg::set_error("sg_blob_size: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_blob_get(sg_net* n, int32_t layer, int32_t which, void* dst_dev, size_t bytes, void* stream) { ::sg::set_error("sg_blob_get: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_blob_set(sg_net* n, int32_t layer, int32_t which, const void* src_dev, size_t bytes,
                             void* stream) { ::sg::set_error("sg_blob_set: not implemented"); return SG_ERR_UNSUPPORTED; }
SG_API sg_status sg_server_sync(sg_cluster* c, const sg_updater_cfg* cfg, int64_t step, float* grad_full_dev,
                                float* w_full_dev, float* v_shard_dev, int64_t n, void* stream) { ::sg::set_error("sg_server_sync: not implemented"); return SG_ERR_UNSUPPORTED; }
}
