// ib_b200/ib/b200.hpp -- plumbing of the drop-in overlay (not a reference
// header): the process-wide device context, status -> exception mapping,
// and the observable workspace results.  Everything here is namespace
// ib::b200; the reference's names live in the sibling headers.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <functional>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ibcuda.h"

namespace ib::b200 {

// Status code -> the reference's exception type (include/ibcuda.h).
inline void check(ibc_status s) {
  switch (s) {
    case IBC_OK:
      return;
    case IBC_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(ibc_last_error());
    case IBC_ERR_LENGTH:
      throw std::length_error(ibc_last_error());
    case IBC_ERR_ALLOC:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(std::string("libibcuda: ") + ibc_last_error());
  }
}

// Device of the process-wide context (set before the first call).
inline int& default_device() {
  static int device = 0;
  return device;
}

// One context per process, created on first use (the reference's implicit
// OpenMP team, parallel.hpp:25-36).
inline ibc_context* context() {
  struct Holder {
    ibc_context* ctx = nullptr;
    ~Holder() {
      if (ctx) ibc_context_destroy(ctx);
    }
  };
  static Holder h;
  if (!h.ctx) check(ibc_context_create(default_device(), &h.ctx));
  return h.ctx;
}

// f(c) for the components c = 0 .. count-1 of a vector operation, one host
// thread each (the calling thread takes the last): the context serves every
// host-buffer call on its own lane (stream, staging, scratch), so the
// components' copies and kernels overlap -- one component's grid download
// beside the next one's upload.  Results do not depend on the overlap.
// Rethrows the lowest component's exception.
template <std::size_t N, class F>
void for_components(std::size_t count, F&& f) {
  context();  // created once, before any thread asks for it
  std::array<std::exception_ptr, N> err{};
  std::vector<std::thread> threads;
  threads.reserve(count);
  for (std::size_t c = 0; c + 1 < count; ++c)
    threads.emplace_back([&f, &err, c] {
      try {
        f(c);
      } catch (...) {
        err[c] = std::current_exception();
      }
    });
  if (count) {
    try {
      f(count - 1);
    } catch (...) {
      err[count - 1] = std::current_exception();
    }
  }
  for (auto& t : threads) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// A workspace result the reference keeps as a plain member (ws.keys,
// ws.perm, ws.run_keys, spread.hpp:33-41).  The device keeps it on the
// device and copies it back on first read after a spread, so a caller that
// never looks pays nothing; reads look like the reference's std::vector.
template <class T>
class observable_vector {
 public:
  using value_type = T;
  using size_type = std::size_t;
  using const_iterator = typename std::vector<T>::const_iterator;

  explicit observable_vector(std::size_t n = 0) : v_(n) {}

  const std::vector<T>& get() const {
    if (stale_ && fill_) {
      fill_(v_);
      stale_ = false;
    }
    return v_;
  }
  operator const std::vector<T>&() const { return get(); }
  operator std::span<const T>() const { return std::span<const T>(get()); }

  const T& operator[](std::size_t i) const { return get()[i]; }
  std::size_t size() const { return v_.size(); }
  bool empty() const { return v_.empty(); }
  const T* data() const { return get().data(); }
  const_iterator begin() const { return get().begin(); }
  const_iterator end() const { return get().end(); }

  friend bool operator==(const observable_vector& a, const std::vector<T>& b) { return a.get() == b; }
  friend bool operator==(const std::vector<T>& b, const observable_vector& a) { return a.get() == b; }

  // Overlay internals: the next read refills from `fill`.
  void invalidate(std::function<void(std::vector<T>&)> fill) {
    fill_ = std::move(fill);
    stale_ = true;
  }

 private:
  mutable std::vector<T> v_;
  mutable bool stale_ = false;
  std::function<void(std::vector<T>&)> fill_;
};

// ws.run_count (spread.hpp:41): q of the most recent spread, read from the
// device on first use.
class observable_count {
 public:
  std::size_t get() const {
    if (stale_ && fill_) {
      v_ = fill_();
      stale_ = false;
    }
    return v_;
  }
  operator std::size_t() const { return get(); }
  friend bool operator==(const observable_count& a, std::size_t b) { return a.get() == b; }
  friend bool operator==(std::size_t b, const observable_count& a) { return a.get() == b; }

  void invalidate(std::function<std::size_t()> fill) {
    fill_ = std::move(fill);
    stale_ = true;
  }

 private:
  mutable std::size_t v_ = 0;
  mutable bool stale_ = false;
  std::function<std::size_t()> fill_;
};

template <class T>
bool operator==(const observable_vector<T>& a, const observable_vector<T>& b) {
  return a.get() == b.get();
}

}  // namespace ib::b200
