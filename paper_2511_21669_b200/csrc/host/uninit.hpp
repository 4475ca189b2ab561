// uninit.hpp — a vector whose resize() leaves trivially constructible
// elements uninitialised (default-init instead of value-init): the planner
// fills million-element replica arrays in parallel, so their first touch -
// the page faults - is spread over the threads instead of a serial zero fill.
#pragma once
#include <memory>
#include <type_traits>
#include <utility>
#include <vector>

namespace dsd::host {

template <class T>
struct default_init_allocator : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = default_init_allocator<U>;
    };
    default_init_allocator() = default;
    template <class U>
    default_init_allocator(const default_init_allocator<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept(std::is_nothrow_default_constructible_v<U>) {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};

template <class T>
using uvector = std::vector<T, default_init_allocator<T>>;

}  // namespace dsd::host
