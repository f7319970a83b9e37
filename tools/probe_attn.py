import torch
s,H,hd=4096,16,128; h=H*hd
qkv=torch.randn(s,3*h,device='cuda',dtype=torch.bfloat16)
v=qkv.view(1,s,3,H,hd); q,k,vv=[v[:,:,i].transpose(1,2) for i in range(3)]
res=torch.ops.aten._scaled_dot_product_cudnn_attention(q,k,vv,None,True,0.0,True,False)
o,lse=res[0],res[1]; meta=res[2:8]
print("o",o.shape,o.stride(),"lse",lse.shape,lse.stride())
do=torch.randn_like(o)
dq,dk,dv=torch.ops.aten._scaled_dot_product_cudnn_attention_backward(do,q,k,vv,o,lse,meta[4],meta[5],None,*meta[:4],0.0,True)
for t in (dq,dk,dv): print(t.shape,t.stride(),t.data_ptr(), t.untyped_storage().nbytes())
print("dk-dq",dk.data_ptr()-dq.data_ptr(),"dv-dk",dv.data_ptr()-dk.data_ptr())
print(dq.transpose(1,2).reshape(s,h).data_ptr()==dq.data_ptr())
