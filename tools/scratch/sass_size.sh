# SASS instruction count of each k_simulate variant in the built library
cuobjdump -sass ${1:-paper_2511_21669_b200/libdsdsim.so} | awk '/Function : /{if(name!="")print n, name; name=$3; n=0} /\/\*[0-9a-f]+\*\/ +[A-Z@]/{n++} END{print n, name}' | grep k_simulate
