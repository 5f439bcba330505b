// Host-side helpers of the upload path that are compiled by g++ (hostcheck.cpp), declared for graph.cu.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <vector>

namespace hsawgpu {

// Pageable -> pinned staging copy (memcpy, or non-temporal stores under HSAW_UPLOAD_NT=1).
void staging_copy(void* dst, const void* src, size_t bytes);

// Do the caller's cumulative weights equal, bit for bit, the 1/in-degree sums the device would
// regenerate from the offsets (indegree_row_cum, graph.cu)? A two-ended work list over row-aligned
// chunks: run()/work() verify chunks from the front, claim_back() hands runs of chunks from the
// back to the uploader, which copies those instead.
class RowCheck {
public:
    RowCheck(uint32_t n, const uint64_t* off, const double* cum, uint64_t edges_per_chunk);
    void run(unsigned threads);  // returns when the list is empty or a row differs
    void work();                 // one worker's loop
    // Claims up to max_chunks unclaimed chunks at the back; [*e0, *e1) is their edge range.
    bool claim_back(uint32_t max_chunks, uint64_t* e0, uint64_t* e1);
    bool differs() const { return differs_.load(); }
    uint64_t checked_edges() const { return checked_.load(); }

private:
    bool claim_front(uint64_t* c);
    uint32_t n_;
    const uint64_t* off_;
    const double* cum_;
    std::vector<uint64_t> rows_;       // chunk c = rows [rows_[c], rows_[c + 1])
    std::atomic<uint64_t> ends_{0};    // front << 32 | back
    std::atomic<bool> differs_{false};
    std::atomic<uint64_t> checked_{0};
    bool avx2_ = false;
};

bool rows_are_indegree_sums(uint32_t n, const uint64_t* off, const double* cum, unsigned threads);

}  // namespace hsawgpu
