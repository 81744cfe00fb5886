// Block-vector handles of the C ABI (block_vector.hpp:53-151): n_rows x n_s
// complex, stored as n_s/n_b device panels, each one cudaMalloc'ed row-major
// n_rows x n_b buffer (the reference's panel layout, block_vector.hpp:49-52), so
// a panel pointer goes straight to the kernels and to peer / IPC mappings.
// swap_blocks (block_vector.hpp:138-141) exchanges panel buffers, O(1).
#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/chebfd_b200.h"
#include "device.hpp"

struct cf_blockvec_s {
    int device = 0;
    std::size_t rows = 0, ns = 0, nb = 0;
    std::vector<void*> panels;
};

namespace {
void check_handle(cf_blockvec v) {
    if (!v) throw std::invalid_argument("null block vector");
}
void check_panel(cf_blockvec v, size_t b) {
    check_handle(v);
    if (b >= v->panels.size()) throw std::out_of_range("panel index out of range");  // block_vector.hpp:107
}
}  // namespace

using namespace cfb;

extern "C" {

int cf_blockvec_create(int device, size_t rows, size_t ns, size_t nb, cf_blockvec* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        *out = nullptr;
        // BlockVector ctor checks (block_vector.hpp:57-66)
        if (nb == 0 || ns == 0 || ns % nb != 0) throw std::invalid_argument("n_b must divide n_s");
        DeviceGuard dg(device);
        auto v = std::make_unique<cf_blockvec_s>();
        v->device = device;
        v->rows = rows;
        v->ns = ns;
        v->nb = nb;
        const std::size_t bytes = rows * nb * 16;
        for (std::size_t b = 0; b < ns / nb; ++b) {
            void* p = nullptr;
            if (bytes) {
                const cudaError_t e = cudaMalloc(&p, bytes);
                if (e != cudaSuccess) {
                    for (void* q : v->panels) cudaFree(q);
                    ck(e, "cudaMalloc block-vector panel");
                }
                ck(cudaMemset(p, 0, bytes), "zero panel");  // InitZero
            }
            v->panels.push_back(p);
        }
        ck(cudaDeviceSynchronize(), "block vector create");
        *out = v.release();
    });
}

int cf_blockvec_destroy(cf_blockvec v) {
    return guard([&] {
        if (!v) return;
        DeviceGuard dg(v->device);
        for (void* p : v->panels) cudaFree(p);
        delete v;
    });
}

int cf_blockvec_shape(cf_blockvec v, size_t* rows, size_t* ns, size_t* nb, int* device) {
    return guard([&] {
        check_handle(v);
        if (rows) *rows = v->rows;
        if (ns) *ns = v->ns;
        if (nb) *nb = v->nb;
        if (device) *device = v->device;
    });
}

int cf_blockvec_panel(cf_blockvec v, size_t b, void** dev_ptr) {
    return guard([&] {
        check_panel(v, b);
        *dev_ptr = v->panels[b];
    });
}

int cf_blockvec_upload(cf_blockvec v, const double* host_panels) {
    return guard([&] {
        check_handle(v);
        DeviceGuard dg(v->device);
        const std::size_t bytes = v->rows * v->nb * 16;
        for (std::size_t b = 0; b < v->panels.size(); ++b)
            if (bytes) ck(cudaMemcpy(v->panels[b], host_panels + 2 * b * v->rows * v->nb, bytes, cudaMemcpyHostToDevice),
                          "upload panel");
    });
}

int cf_blockvec_download(cf_blockvec v, double* host_panels) {
    return guard([&] {
        check_handle(v);
        DeviceGuard dg(v->device);
        const std::size_t bytes = v->rows * v->nb * 16;
        ck(cudaDeviceSynchronize(), "block vector download");
        for (std::size_t b = 0; b < v->panels.size(); ++b)
            if (bytes) ck(cudaMemcpy(host_panels + 2 * b * v->rows * v->nb, v->panels[b], bytes, cudaMemcpyDeviceToHost),
                          "download panel");
    });
}

int cf_panel_swap(cf_blockvec a, size_t ia, cf_blockvec b, size_t ib) {
    return guard([&] {
        check_panel(a, ia);
        check_panel(b, ib);
        // swap_blocks (block_vector.hpp:138-146): same shape, same device
        if (a->rows != b->rows || a->nb != b->nb) throw std::invalid_argument("swap_blocks: shape mismatch");
        if (a->device != b->device) throw std::invalid_argument("swap_blocks: panels on different devices");
        std::swap(a->panels[ia], b->panels[ib]);
    });
}

}  // extern "C"
